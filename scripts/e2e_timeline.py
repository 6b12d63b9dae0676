"""Timeline of the e2e step (public API on pinned host buffers): A upload, detection, then per B
column slab its upload, its SpMM and its C download, as event timestamps on each stream, next to
the PCIe floor. Same calls as executor._run_host_pipelined, with events in between.
   python scripts/e2e_timeline.py [slabs]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2301_10936_b200 as pit  # noqa: E402
from paper_2301_10936_b200 import _lib  # noqa: E402
from paper_2301_10936_b200.executor import spmm_device  # noqa: E402

dev = torch.device("cuda", 0)
w = dict(bench.WORKLOADS["pitk_c1_8192"], name="pitk_c1_8192")
A, B, live = bench.make_operands(w, 1234, dev)
plan = bench.make_plan(w)
Ah = torch.empty(A.t().shape, dtype=A.dtype, pin_memory=True)
Ah.copy_(A.t())
Bh = torch.empty(B.shape, dtype=B.dtype, pin_memory=True)
Bh.copy_(B)
del A, B
lib = _lib.load()
main = torch.cuda.current_stream()
s_up, s_down = torch.cuda.Stream(), torch.cuda.Stream()
K, N = Bh.shape
M = Ah.shape[1]
eb = 2
Bd = torch.empty((K, N), dtype=Bh.dtype, device=dev)
Cd = torch.empty((M, N), dtype=Bh.dtype, device=dev)
Ch = torch.empty((M, N), dtype=Bh.dtype, pin_memory=True)
Ad = torch.empty(Ah.shape, dtype=Ah.dtype, device=dev)


def ev(s):
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    return e


def step(sched):
    marks = []
    t0 = ev(main)
    Ad.copy_(Ah, non_blocking=True)
    marks.append(("A up", ev(main)))
    idx = pit.build_index_from_tensor(Ad.t(), w["micro"], w["axis"])
    marks.append(("detect", ev(main)))
    starts = [sum(sched[:i]) for i in range(len(sched))]
    s_up.wait_stream(main)
    ups = []
    for j0, slab in zip(starts, sched):
        with torch.cuda.stream(s_up):
            lib.pit_copy2d_async(Bd.data_ptr() + j0 * eb, N * eb, Bh.data_ptr() + j0 * eb, N * eb, slab * eb, K,
                                 s_up.cuda_stream)
            ups.append(ev(s_up))
    for i, (j0, slab) in enumerate(zip(starts, sched)):
        main.wait_event(ups[i])
        spmm_device(plan, Ad.t(), Bd[:, j0:j0 + slab], idx, out=Cd[:, j0:j0 + slab])
        ec = ev(main)
        s_down.wait_event(ec)
        with torch.cuda.stream(s_down):
            lib.pit_copy2d_async(Ch.data_ptr() + j0 * eb, N * eb, Cd.data_ptr() + j0 * eb, N * eb, slab * eb, M,
                                 s_down.cuda_stream)
            ed = ev(s_down)
        marks.append((f"slab {i}: up {t0.elapsed_time(ups[i]) if False else 0}", (ups[i], ec, ed)))
    main.wait_stream(s_down)
    end = ev(main)
    torch.cuda.synchronize()
    out = [f"  A up {t0.elapsed_time(marks[0][1]):7.3f}  detect {t0.elapsed_time(marks[1][1]):7.3f}"]
    for i, (_, (u, c, d)) in enumerate(marks[2:]):
        out.append(f"  slab {i:2d}: up done {t0.elapsed_time(u):7.3f}  spmm done {t0.elapsed_time(c):7.3f}  "
                   f"down done {t0.elapsed_time(d):7.3f}")
    return t0.elapsed_time(end), out


for arg in sys.argv[1:] or ["[1024]*8"]:
    sched = [int(x) for x in (eval(arg) if arg.startswith("[") else arg.split(","))]  # "[1024]*8" or "512,..."
    assert sum(sched) == N, (arg, sum(sched))
    for _ in range(2):
        step(sched)
    tots = []
    for _ in range(3):
        tot, lines = step(sched)
        tots.append(tot)
    print(f"slabs {arg}: step {min(tots):.3f} ms (of {', '.join(f'{t:.3f}' for t in tots)})")
    print("\n".join(lines))
