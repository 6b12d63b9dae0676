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

    def pack_groups(self, src, rows, stride, counts, offsets, max_count, n_rows):
        """csrc pack_groups_kernel: out[offsets[g] + i] = src[rows[g, i]] for i < counts[g]."""
        out = src.new_zeros((max(n_rows, 1), src.shape[1]))
        for g in range(counts.numel()):
            c, o = int(counts[g]), int(offsets[g])
            out[o:o + c] = src[rows.view(-1, stride)[g, :c].long()]
        return out

    def scatter_rows_scaled(self, src, rows, n, scale, out):
        r = rows[:n].long()
        out[r] = (src[:n].double() * scale[r].double()[:, None]).to(out.dtype)
        return out

    def grouped_gemm(self, A, W, counts, offsets, tiles, out, *, row_src=None, src_stride=0, row_dst=None,
                     dst_stride=0, row_scale=None, act=0, max_tiles=None, rows_hint=0):
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


class EmulatedPeerExchange:
    """CPU restatement of the peer-memory exchange protocol of csrc/pit_ep.cu over gloo.

    Same region layout and row positions as the kernels: source rank s's rows for rank r land in
    r's receive region at s * cap + (position among the tokens s sends to r, in expert order); the
    per-expert counts land in r's counts[s]; the receive plan lists a local expert's rows in
    source-rank order; combine pulls row rank * cap + position from the expert rank's y region.
    A store into a peer region is emulated by all_to_all_single of the padded per-peer slabs."""

    def __init__(self, group, experts_local, capacity, d_model, dtype, device=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.El, self.cap, self.d_model = experts_local, capacity, d_model
        R = self.world * self.cap
        self.recv = torch.zeros((R, d_model), dtype=dtype)
        self.y = torch.zeros((R, d_model), dtype=dtype)
        self.counts_in = torch.zeros((self.world, self.El), dtype=torch.int32)
        self.rows = torch.zeros((self.El, max(R, 1)), dtype=torch.int32)
        self.lcounts = torch.zeros(self.El, dtype=torch.int32)
        self._pulled = None

    def _a2a(self, send):
        import torch.distributed as dist

        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send.contiguous(), group=self.group)
        return recv

    def dispatch(self, x, perm, offsets, counts):
        W, El, cap = self.world, self.El, self.cap
        off = offsets.numpy()
        slab = torch.zeros((W, cap, self.d_model), dtype=x.dtype)
        for i in range(int(off[-1])):
            e = int(np.searchsorted(off, i, side="right") - 1)
            r = e // El
            slab[r, i - off[r * El]] = x[int(perm[i])]
        got = self._a2a(slab)  # got[s] = what rank s stored into my region
        for s in range(W):
            self.recv[s * cap:(s + 1) * cap] = got[s]
        self.counts_in = self._a2a(counts.view(W, El).to(torch.int32))

    def recv_plan(self):
        rc = self.counts_in.numpy()
        for e in range(self.El):
            out = 0
            for s in range(self.world):
                before, n = int(rc[s, :e].sum()), int(rc[s, e])
                self.rows[e, out:out + n] = torch.arange(s * self.cap + before, s * self.cap + before + n)
                out += n
            self.lcounts[e] = out
        return self.rows, self.lcounts

    def signal(self):
        # peer s will pull rows [s*cap, (s+1)*cap) of my y: emulate the pull by sending that slab
        self._pulled = self._a2a(self.y.view(self.world, self.cap, self.d_model))

    def combine(self, perm, offsets, gate, out):
        off = offsets.numpy()
        for i in range(int(off[-1])):
            e = int(np.searchsorted(off, i, side="right") - 1)
            r = e // self.El
            t = int(perm[i])
            g = float(gate[t]) if gate is not None else 1.0
            out[t] = (self._pulled[r, i - off[r * self.El]].double() * g).to(out.dtype)
        return out

    def error(self):
        return 0

    def close(self):
        pass
