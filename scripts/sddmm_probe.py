"""C3 attention-score SDDMM at full size: per-launch device times of index build vs the kernel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2301_10936_b200 as pit
from paper_2301_10936_b200.sddmm import output_indexes, run_batched_sddmm

import os
heads, seq, hd = int(os.environ.get("H", 12)), int(os.environ.get("S", 4096)), 64
rng = np.random.default_rng(3)
qi = np.arange(seq // 32)[:, None] * 32 + 16
kj = np.arange(seq // 64)[None, :] * 64 + 32
base = np.abs(qi - kj) <= 256 + 48
base[:, 0] = True
base[0, :] = True
blocks = np.stack([base | (rng.random(base.shape) < 0.02) for _ in range(heads)])
ann = pit.from_bits(blocks.reshape(heads * seq // 32, seq // 64), (heads * seq, seq), (32, 64)).on_device(torch.device("cuda"))
g = torch.Generator(device="cuda").manual_seed(5)
Q = torch.randn((heads, seq, hd), device="cuda", dtype=torch.bfloat16, generator=g)
Kt = torch.randn((heads, seq, hd), device="cuda", dtype=torch.bfloat16, generator=g)
S = torch.zeros((heads, seq, seq), device="cuda", dtype=torch.bfloat16)
idx = output_indexes(ann)
for _ in range(3):
    run_batched_sddmm(Q, Kt.transpose(1, 2), ann, out=S, indexes=idx)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ts = []
for _ in range(10):
    e[0].record()
    ix = output_indexes(ann)
    e[1].record()
    run_batched_sddmm(Q, Kt.transpose(1, 2), ann, out=S, indexes=ix)
    e[2].record()
    torch.cuda.synchronize()
    ts.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
print("index ms %.4f  sddmm ms %.4f" % tuple(np.median(np.array(ts), axis=0)))
print("units", int(sum(-(-c // 4) for c in idx[0].counts)), "groups", idx[0].n_groups, "live blocks", int(blocks.sum()))
