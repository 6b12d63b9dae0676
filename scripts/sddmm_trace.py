"""Unit timeline of the SDDMM kernel (CTA 0) from PIT_SD_DIAG bit 4 stamps (diagnostic build:
PIT_DIAG=1 scripts/build_alt.sh WT diag; PIT_LIB_PATH=build_alt/libpit_diag.so PIT_SD_DIAG=16 python scripts/sddmm_trace.py)."""
import ctypes
import os
import runpy
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
runpy.run_path(str(Path(__file__).resolve().parent / "sddmm_probe.py"))
from paper_2301_10936_b200 import _lib  # noqa: E402

buf = (ctypes.c_ulonglong * 512)()
_lib.load().pit_debug_sddmm_trace(buf)
t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(8, 64)
t0 = t[t > 0].min()
names = ["P meta", "P tma", "M full", "M commit", "E meta", "E tfull", "E end4", "E end11"]
print("unit " + " ".join(f"{n:>9s}" for n in names) + "   (ns from CTA 0's first stamp)")
for u in range(64):
    if t[:, u].max() == 0:
        break
    print(f"{u:4d} " + " ".join(f"{(x - t0) if x else -1:9d}" for x in t[:, u]))
