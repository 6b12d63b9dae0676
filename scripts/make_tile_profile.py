"""Profile every registered tile on this B200 (tiles.profile, CUDA events) and save the table in the
reference's `pit-profile v1` format (profiles/<round>/b200_tiles.prof)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2301_10936_b200 as pit  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/b200_tiles.prof"
table = pit.profile(pit.register_builtin_kernels(include_b200_tiles=True), reps=3)
pit.save_profile(table, out)
print(open(out).read())
