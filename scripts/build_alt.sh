#!/bin/bash
# Build libpit_b200.so of git revision REV (or the working tree: REV=WT) into build_alt/libpit_NAME.so
# for same-box A/B timing (PIT_LIB_PATH=build_alt/libpit_NAME.so). Extra -D flags: PIT_NVCC_DEFS.
#   scripts/build_alt.sh REV [NAME]
set -e
REV=${1:-HEAD}
NAME=${2:-$REV}
TMP=$(mktemp -d)
if [ "$REV" = WT ]; then
  mkdir -p "$TMP/paper_2301_10936_b200"
  cp -r paper_2301_10936_b200/csrc paper_2301_10936_b200/_build.py "$TMP/paper_2301_10936_b200/"
  cp -r include "$TMP/"
else
  git archive "$REV" paper_2301_10936_b200/csrc paper_2301_10936_b200/_build.py include | tar -x -C "$TMP"
fi
(cd "$TMP" && python paper_2301_10936_b200/_build.py --force > /dev/null)
mkdir -p build_alt
cp "$TMP/paper_2301_10936_b200/libpit_b200.so" "build_alt/libpit_$NAME.so"
rm -rf "$TMP"
echo "build_alt/libpit_$NAME.so"
