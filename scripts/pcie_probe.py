"""Host<->device copy rates on this box: contiguous and pitched (column-slab) H2D / D2H, alone and
overlapped (the e2e path's ceilings)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2301_10936_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
n = 8192
h = torch.empty((n, n), dtype=torch.bfloat16, pin_memory=True)
d = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
h2 = torch.empty((n, n), dtype=torch.bfloat16, pin_memory=True)
d2 = torch.empty((n, n), dtype=torch.bfloat16, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nbytes = n * n * 2


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def slabs(dst, src, up, stream, slab=1024):
    for j0 in range(0, n, slab):
        lib.pit_copy2d_async(dst.data_ptr() + j0 * 2, n * 2, src.data_ptr() + j0 * 2, n * 2, slab * 2, n,
                             stream.cuda_stream)


ms = timed(lambda: d.copy_(h, non_blocking=True))
print(f"H2D contiguous 128 MiB: {ms:.3f} ms = {nbytes / ms / 1e6:.1f} GB/s")
ms = timed(lambda: h.copy_(d, non_blocking=True))
print(f"D2H contiguous 128 MiB: {ms:.3f} ms = {nbytes / ms / 1e6:.1f} GB/s")
cur = torch.cuda.current_stream()
ms = timed(lambda: slabs(d, h, True, cur))
print(f"H2D 1024-column slabs: {ms:.3f} ms = {nbytes / ms / 1e6:.1f} GB/s")
ms = timed(lambda: slabs(h, d, False, cur))
print(f"D2H 1024-column slabs: {ms:.3f} ms = {nbytes / ms / 1e6:.1f} GB/s")


def both():
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ms = timed(both)
print(f"H2D + D2H concurrent (128 MiB each): {ms:.3f} ms = {2 * nbytes / ms / 1e6:.1f} GB/s total")


def two_up():
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ms = timed(two_up)
print(f"2x H2D concurrent (128 MiB each): {ms:.3f} ms = {2 * nbytes / ms / 1e6:.1f} GB/s total")
