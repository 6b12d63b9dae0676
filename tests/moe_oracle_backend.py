"""Test-only MoE backend: the oracle's arithmetic on CPU torch tensors, so the expert-parallel
orchestration of paper_2301_10936_b200.moe.SwitchMoE can run over gloo without a GPU.
Not part of the product (the product backend is CudaBackend)."""

import numpy as np
import torch

from oracle import pit_oracle as orc


class OracleBackend:
    def route(self, logits):
        expert, gate, counts, groups = orc.switch_route(logits.float().numpy())
        T, E = logits.shape
        slots = np.zeros((E, max(T, 1)), np.int32)
        for e, g in enumerate(groups):
            slots[e, : g.size] = g
        return (torch.from_numpy(expert.astype(np.int32)), torch.from_numpy(gate.astype(np.float32)),
                torch.from_numpy(counts.astype(np.int32)), torch.from_numpy(slots))

    def plan(self, counts, slots=None, stride=0, total=0):
        c = counts.numpy().astype(np.int64)
        offsets = np.concatenate([[0], np.cumsum(c)]).astype(np.int32)
        tiles = np.concatenate([[0], np.cumsum(-(-c // 128))]).astype(np.int32)
        perm = None
        if slots is not None:
            perm = torch.from_numpy(np.concatenate([slots.numpy()[g, : c[g]] for g in range(len(c))] or
                                                   [np.zeros(0, np.int32)]).astype(np.int32))
        return torch.from_numpy(offsets), torch.from_numpy(tiles), perm

    def recv_plan(self, rc, R):
        rc = rc.numpy()
        W, El = rc.shape
        rows = np.zeros((El, max(R, 1)), np.int32)
        counts = rc.sum(axis=0).astype(np.int32)
        base = np.concatenate([[0], np.cumsum(rc.sum(axis=1))])
        for e in range(El):
            out = []
            for r in range(W):
                start = base[r] + rc[r, :e].sum()
                out.extend(range(start, start + rc[r, e]))
            rows[e, : len(out)] = out
        return torch.from_numpy(rows), torch.from_numpy(counts)

    def gather_rows(self, src, rows, n):
        return src[rows[:n].long()].clone()

    def scatter_rows_scaled(self, src, rows, n, scale, out):
        r = rows[:n].long()
        out[r] = (src[:n].double() * scale[r].double()[:, None]).to(out.dtype)
        return out

    def grouped_gemm(self, A, W, counts, offsets, tiles, out, *, row_src=None, src_stride=0, row_dst=None,
                     dst_stride=0, row_scale=None, act=0, max_tiles=None):
        for g in range(W.shape[0]):
            c, o = int(counts[g]), int(offsets[g])
            if c == 0:
                continue
            src = row_src[g, :c].long() if row_src is not None else torch.arange(o, o + c)
            dst = row_dst[g, :c].long() if row_dst is not None else torch.arange(o, o + c)
            y = A[src].double() @ W[g].double()
            if act == 1:
                y = y.clamp_min(0.0)
            if row_scale is not None:
                y = y * row_scale[dst].double()[:, None]
            out[dst] = y.to(out.dtype)
        return out
