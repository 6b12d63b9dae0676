#!/bin/bash
# Build libpit_b200.so of git revision REV into build_alt/libpit_REV.so (A/B timing against the
# working tree on the same box: PIT_LIB_PATH=build_alt/libpit_REV.so).
set -e
REV=${1:-HEAD}
TMP=$(mktemp -d)
git archive "$REV" paper_2301_10936_b200/csrc paper_2301_10936_b200/_build.py include | tar -x -C "$TMP"
(cd "$TMP" && python paper_2301_10936_b200/_build.py --force > /dev/null)
mkdir -p build_alt
cp "$TMP/paper_2301_10936_b200/libpit_b200.so" "build_alt/libpit_$REV.so"
rm -rf "$TMP"
echo "build_alt/libpit_$REV.so"
