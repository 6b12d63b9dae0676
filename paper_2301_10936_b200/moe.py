"""Switch-style MoE layer (top-1, dropless) on the PIT path, with expert parallelism.

PIT's view of an MoE layer: the router produces a [T, E]
one-hot mask whose PIT index (groups = experts, coordinates = tokens) is built online; the expert
FFNs are per-expert gathered-row GEMMs (SRead of the token rows fused into the mainloop), and the
combine is an SWrite scaled by the gate. No capacity padding: every token is computed once.

Expert parallelism over W ranks (rank r owns experts [r*E/W, (r+1)*E/W)), two exchanges:
  "peer" (the product, `PeerExchange`): route -> plan -> dispatch (SRead pack fused with the send:
      token rows stored straight into the owning rank's receive region over NVLink) -> receive
      plan (waits on the peers' epoch flags) -> FFN1 (ReLU) -> FFN2 (into the y region) -> signal
      -> combine (each token pulls its output row from the expert rank, SWrite * gate fused).
      No host synchronisation: the whole layer is capturable in one CUDA graph.
  "nccl" (baseline): pack -> all_to_all(counts) -> one D2H of the split sizes -> all_to_all_v(tokens)
      -> receive plan -> FFN1 -> FFN2 -> all_to_all_v(back) -> combine.
The orchestration is written against a backend: `CudaBackend` (libpit_b200.so kernels) is the
product; the NCCL-path exchange logic is backend-agnostic so it can be exercised over gloo in tests.
"""

from __future__ import annotations

import os

import ctypes as C
from dataclasses import dataclass
from typing import Optional

from . import _device, _lib


def _torch():
    import torch

    return torch


class CudaBackend:
    """Device kernels for the MoE path (all tensors on the current CUDA device)."""

    def __init__(self):
        self.lib = _lib.load()

    def _stream(self):
        return _device.stream_ptr()

    def route(self, logits):
        torch = _torch()
        T, E = logits.shape
        dev = logits.device
        expert = torch.empty(T, dtype=torch.int32, device=dev)
        gate = torch.empty(T, dtype=torch.float32, device=dev)
        occ = torch.empty(E * max(1, -(-T // 32)), dtype=torch.int32, device=dev)
        counts = torch.empty(E, dtype=torch.int32, device=dev)
        slots = torch.empty((E, max(T, 1)), dtype=torch.int32, device=dev)
        logits = logits.contiguous()
        _device.check(self.lib.pit_moe_route(logits.data_ptr(), _device.dtype_code(logits), T, E, expert.data_ptr(),
                                             gate.data_ptr(), occ.data_ptr(), counts.data_ptr(), slots.data_ptr(),
                                             self._stream()))
        return expert, gate, counts, slots

    def plan(self, counts, slots=None, stride=0, total=0):
        torch = _torch()
        G = counts.numel()
        dev = counts.device
        offsets = torch.empty(G + 1, dtype=torch.int32, device=dev)
        tiles = torch.empty(G + 1, dtype=torch.int32, device=dev)
        perm = torch.empty(max(total, 1), dtype=torch.int32, device=dev) if slots is not None else None
        _device.check(self.lib.pit_moe_plan(counts.data_ptr(), G, slots.data_ptr() if slots is not None else None,
                                            stride, offsets.data_ptr(), tiles.data_ptr(),
                                            perm.data_ptr() if perm is not None else None, max(total, 1),
                                            self._stream()))
        return offsets, tiles, perm

    def recv_plan(self, rc, R):
        torch = _torch()
        W, El = rc.shape
        rows = torch.empty((El, max(R, 1)), dtype=torch.int32, device=rc.device)
        counts = torch.empty(El, dtype=torch.int32, device=rc.device)
        rc = rc.to(torch.int32).contiguous()
        _device.check(self.lib.pit_moe_recv_plan(rc.data_ptr(), W, El, rows.data_ptr(), max(R, 1), counts.data_ptr(),
                                                 self._stream()))
        return rows, counts

    def gather_rows(self, src, rows, n):
        torch = _torch()
        out = torch.empty((n, src.shape[1]), dtype=src.dtype, device=src.device)
        eb = src.element_size()
        _device.check(self.lib.pit_gather_rows(src.data_ptr(), src.stride(0) * eb, rows.data_ptr(), n,
                                               src.shape[1] * eb, out.data_ptr(), out.stride(0) * eb, self._stream()))
        return out

    def pack_groups(self, src, rows, stride, counts, offsets, max_count, n_rows):
        """Group-wise SRead: row offsets[g] + i of the result = src row rows[g * stride + i]."""
        torch = _torch()
        out = torch.empty((max(n_rows, 1), src.shape[1]), dtype=src.dtype, device=src.device)
        eb = src.element_size()
        _device.check(self.lib.pit_pack_groups(src.data_ptr(), src.stride(0) * eb, rows.data_ptr(), stride,
                                               counts.data_ptr(), offsets.data_ptr(), counts.numel(), max_count,
                                               src.shape[1] * eb, out.data_ptr(), out.stride(0) * eb, self._stream()))
        return out

    def scatter_rows_scaled(self, src, rows, n, scale, out):
        _device.check(self.lib.pit_scatter_rows_scaled(src.data_ptr(), _device.dtype_code(src), src.stride(0),
                                                       rows.data_ptr(), n, src.shape[1],
                                                       scale.data_ptr() if scale is not None else None,
                                                       out.data_ptr(), out.stride(0), self._stream()))
        return out

    def grouped_gemm(self, A, W, counts, offsets, tiles, out, *, row_src=None, src_stride=0, row_dst=None,
                     dst_stride=0, row_scale=None, act=0, max_tiles=None, rows_hint=0):
        G, K, N = W.shape
        a = _lib.GroupedGemmArgs()
        a.dtype = _device.dtype_code(A)
        a.A, a.lda, a.rows_a = A.data_ptr(), A.stride(0), A.shape[0]
        a.B, a.ldb = W.data_ptr(), W.stride(1)
        a.C, a.ldc = out.data_ptr(), out.stride(0)
        a.N, a.K, a.G = N, K, G
        a.counts, a.offsets, a.tile_offsets = counts.data_ptr(), offsets.data_ptr(), tiles.data_ptr()
        a.row_src = row_src.data_ptr() if row_src is not None else None
        a.src_stride = src_stride
        a.row_dst = row_dst.data_ptr() if row_dst is not None else None
        a.dst_stride = dst_stride
        a.row_scale = row_scale.data_ptr() if row_scale is not None else None
        a.act = act
        a.max_tiles = max_tiles if max_tiles is not None else -(-A.shape[0] // 128) + G
        a.rows_hint = rows_hint
        _device.check(self.lib.pit_grouped_gemm(C.byref(a), self._stream()))
        return out


def _raw_view(ptr: int, rows: int, cols: int, dtype, device):
    """Zero-copy torch view [rows, cols] of raw device memory (a region allocated by the C library)."""
    torch = _torch()
    elem = torch.empty((), dtype=dtype).element_size()
    carrier = {2: "<i2", 4: "<i4", 8: "<i8"}[elem]

    class _CAI:
        __cuda_array_interface__ = {"shape": (rows, cols), "typestr": carrier, "data": (ptr, False), "version": 3,
                                    "strides": None}

    raw = torch.as_tensor(_CAI(), device=device)
    return raw.view(dtype)


# FFN1's tokens are packed into expert order first (one group-wise SRead, pit_pack_groups), so the
# grouped GEMM reads its A rows by TMA instead of cp.async row gathers: EP8 per-rank proxy (16 experts
# x ~1024 tokens, CTA-pair tiles) 0.220 -> 0.191 ms; 128-expert layer (~128 tokens per expert,
# swapped-role kernel) 0.302 -> 0.290 ms (CUDA-graph timing). PIT_MOE_PACK=0 gathers instead (A/B knob).
_PACK_ENV = os.environ.get("PIT_MOE_PACK")


def _pack_ffn1(rows_hint: int, groups: int) -> bool:
    return _PACK_ENV != "0"


class PeerUnavailable(RuntimeError):
    """Some rank of the group cannot map the others' exchange regions (no CUDA IPC / peer access).
    Raised on every rank together."""


class PeerExchange:
    """One exchange region per rank, mapped into every other rank through CUDA IPC (pit_ep_* in the C
    ABI). `dispatch` / `recv_plan` / `signal` / `combine` are stream-ordered device calls with no host
    synchronisation. `capacity` = the most tokens a rank sends per layer.

    Collective: every rank of `group` constructs it (and closes it) together."""

    def __init__(self, group, experts_local: int, capacity: int, d_model: int, dtype, device=None):
        import torch.distributed as dist

        torch = _torch()
        self.lib = _lib.load()
        self.group = group
        self.world = dist.get_world_size(group) if group is not None else 1
        self.rank = dist.get_rank(group) if group is not None else 0
        self.El, self.cap, self.d_model, self.dtype = int(experts_local), int(capacity), int(d_model), dtype
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        elem = torch.empty((), dtype=dtype).element_size()
        self.row_bytes = self.d_model * elem
        lay = (C.c_int64 * 6)()
        _device.check(self.lib.pit_ep_region_layout(self.world, self.El, self.cap, self.row_bytes, lay))
        self.layout = dict(zip(("flags_d", "flags_c", "counts", "recv", "y", "total"), list(lay)))
        region = C.c_void_p()
        _device.check(self.lib.pit_ep_region_alloc(self.layout["total"], C.byref(region)))
        self.region = region.value
        self._opened = []
        peers = [0] * self.world
        peers[self.rank] = self.region
        if self.world > 1:
            # every rank learns whether every rank mapped every peer: a rank whose IPC open fails must
            # not leave the others waiting in the barrier below (they all raise PeerUnavailable)
            err = ""
            h = (C.c_char * 64)()
            if self.lib.pit_ep_ipc_handle(self.region, h) != 0:
                err = _lib.last_error()
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(h) if not err else None, group=group)
            for r in range(self.world):
                if r == self.rank or err:
                    continue
                if handles[r] is None:
                    err = f"rank {r} could not export its region"
                    break
                p = C.c_void_p()
                if self.lib.pit_ep_ipc_open(C.create_string_buffer(handles[r], 64), C.byref(p)) != 0:
                    err = f"opening rank {r}'s region: {_lib.last_error()}"
                    break
                self._opened.append(p.value)
                peers[r] = p.value
            errs = [None] * self.world
            dist.all_gather_object(errs, err, group=group)
            bad = [(r, e) for r, e in enumerate(errs) if e]
            if bad:
                for q in self._opened:
                    self.lib.pit_ep_ipc_close(q)
                self._opened = []
                self.lib.pit_ep_region_free(self.region)
                self.region = None
                raise PeerUnavailable(f"peer-memory exchange unavailable (rank {bad[0][0]}: {bad[0][1]})")
        self.peers_dev = torch.tensor(peers, dtype=torch.int64, device=self.device)
        self.args = _lib.EpArgs(self.rank, self.world, self.El, self.cap, self.row_bytes, self.region,
                                self.peers_dev.data_ptr())
        rows_total = self.world * self.cap
        self.recv = _raw_view(self.region + self.layout["recv"], rows_total, self.d_model, dtype, self.device)
        self.y = _raw_view(self.region + self.layout["y"], rows_total, self.d_model, dtype, self.device)
        self.rows = torch.empty((self.El, max(rows_total, 1)), dtype=torch.int32, device=self.device)
        self.lcounts = torch.empty(self.El, dtype=torch.int32, device=self.device)
        if self.world > 1:
            torch.cuda.synchronize(self.device)
            dist.barrier(group)  # every rank mapped every region before anyone writes

    def _s(self):
        return _device.stream_ptr()

    def dispatch(self, x, perm, offsets, counts):
        _device.check(self.lib.pit_moe_dispatch(C.byref(self.args), x.data_ptr(), x.stride(0) * x.element_size(),
                                                x.shape[0], perm.data_ptr(), offsets.data_ptr(), counts.data_ptr(),
                                                self._s()))

    def recv_plan(self):
        _device.check(self.lib.pit_moe_recv_plan_ep(C.byref(self.args), self.rows.data_ptr(), self.rows.shape[1],
                                                    self.lcounts.data_ptr(), self._s()))
        return self.rows, self.lcounts

    def signal(self):
        _device.check(self.lib.pit_moe_signal(C.byref(self.args), self._s()))

    def combine(self, perm, offsets, gate, out):
        _device.check(self.lib.pit_moe_combine(C.byref(self.args), _device.dtype_code(out), out.shape[0],
                                               perm.data_ptr(), offsets.data_ptr(),
                                               gate.data_ptr() if gate is not None else None, out.data_ptr(),
                                               out.stride(0) * out.element_size(), self._s()))
        return out

    def error(self) -> int:
        v = C.c_int()
        _device.check(self.lib.pit_ep_error(self.region, C.byref(v)))
        return v.value

    def close(self):
        """Collective: unmap the peers' regions and free this rank's."""
        if self.region is None:
            return
        torch = _torch()
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier(self.group)  # nobody still reads or writes a region
        for p in self._opened:
            self.lib.pit_ep_ipc_close(p)
        self._opened = []
        self.recv = self.y = None
        self.lib.pit_ep_region_free(self.region)
        self.region = None


@dataclass
class MoEStats:
    tokens: int = 0
    sent: int = 0
    received: int = 0


class SwitchMoE:
    """Top-1 Switch FFN layer: out[t] = gate[t] * W2_e(relu(W1_e x[t])), e = argmax(logits[t]).

    w1: [E_local, d_model, d_ff], w2: [E_local, d_ff, d_model] (bf16/fp16, the rank's experts).
    With a process group of W ranks, E = W * E_local and tokens are exchanged with all-to-all.
    """

    def __init__(self, w1, w2, n_experts: int, group=None, backend=None, exchange: Optional[str] = None,
                 capacity: Optional[int] = None, exchange_factory=None):
        torch = _torch()
        self.w1 = w1.contiguous()
        self.w2 = w2.contiguous()
        self.E = int(n_experts)
        self.El = int(w1.shape[0])
        self.d_model = int(w1.shape[1])
        self.d_ff = int(w1.shape[2])
        self.group = group
        if group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        if self.El * self.world != self.E:
            raise ValueError(f"{self.E} experts do not split over {self.world} ranks of {self.El}")
        if tuple(w2.shape) != (self.El, self.d_ff, self.d_model):
            raise ValueError(f"w2 shape {tuple(w2.shape)} does not match w1 {tuple(w1.shape)}")
        self.backend = backend if backend is not None else CudaBackend()
        self.stats = MoEStats()
        self._torch = torch
        # "peer": device-driven exchange over NVLink (default with W > 1); "nccl": all-to-all-v baseline;
        # "local": single-GPU path (W == 1). "peer" at W == 1 runs the exchange kernels against itself.
        self.exchange = exchange or ("local" if self.world == 1 else "peer")
        self._exchange_requested = exchange is not None
        self.fallback_reason = None
        if self.exchange not in ("local", "peer", "nccl"):
            raise ValueError(f"unknown exchange {self.exchange!r}")
        if self.exchange == "local" and self.world > 1:
            raise ValueError("the local path runs on one rank")
        self.capacity = capacity
        self._peer = None
        self._peer_factory = exchange_factory or PeerExchange

    # --------------------------------------------------------------------------- forward
    def forward(self, x, logits):
        if self.exchange == "local":
            return self._forward_local(x, logits)
        if self.exchange == "peer":
            return self._forward_peer(x, logits)
        return self._forward_ep(x, logits)

    def close(self):
        if self._peer is not None:
            self._peer.close()
            self._peer = None

    def _forward_peer(self, x, logits):
        torch = self._torch
        be = self.backend
        T = x.shape[0]
        if self._peer is None:  # collective: the first call of every rank creates the regions
            cap = self.capacity if self.capacity is not None else T
            try:
                self._peer = self._peer_factory(self.group, self.El, cap, self.d_model, x.dtype, x.device)
            except PeerUnavailable as e:
                if self._exchange_requested:
                    raise
                # default exchange on a box without peer mappings: every rank switches to the NCCL
                # all-to-all-v exchange together (the error was raised on all of them)
                self.exchange, self.fallback_reason = "nccl", str(e)
                return self._forward_ep(x, logits)
        ex = self._peer
        if T > ex.cap:
            raise ValueError(f"{T} tokens exceed the exchange capacity {ex.cap}")
        expert, gate, counts, slots = be.route(logits)
        offsets, _, perm = be.plan(counts, slots, slots.shape[1], T)
        ex.dispatch(x, perm, offsets, counts)               # SRead pack + send over NVLink
        rows, lcounts = ex.recv_plan()                      # waits for every peer's tokens
        loff, ltiles, _ = be.plan(lcounts)
        R = self.world * ex.cap
        h = torch.empty((R, self.d_ff), dtype=x.dtype, device=x.device)
        max_tiles = -(-R // 128) + self.El
        if _pack_ffn1(T, self.El):  # the received tokens in local-expert order, read by TMA
            xp = be.pack_groups(ex.recv, rows, rows.shape[1], lcounts, loff, rows.shape[1], R)
            be.grouped_gemm(xp, self.w1, lcounts, loff, ltiles, h, act=1, max_tiles=max_tiles, rows_hint=T)
        else:
            be.grouped_gemm(ex.recv, self.w1, lcounts, loff, ltiles, h, row_src=rows, src_stride=rows.shape[1],
                            act=1, max_tiles=max_tiles, rows_hint=T)
        be.grouped_gemm(h, self.w2, lcounts, loff, ltiles, ex.y, row_dst=rows, dst_stride=rows.shape[1],
                        max_tiles=max_tiles, rows_hint=T)
        ex.signal()                                         # y ready for the peers' pulls
        out = torch.empty((T, self.d_model), dtype=x.dtype, device=x.device)
        ex.combine(perm, offsets, gate, out)                # pull + SWrite * gate
        self.stats = MoEStats(tokens=T, sent=T, received=-1)
        return out

    __call__ = forward

    def _forward_local(self, x, logits):
        torch = self._torch
        be = self.backend
        T = x.shape[0]
        expert, gate, counts, slots = be.route(logits)
        h = torch.empty((T, self.d_ff), dtype=x.dtype, device=x.device)
        if _pack_ffn1(T, self.E):
            # SRead the tokens into expert order first: FFN1 then reads its A rows by TMA
            offsets, tiles, _ = be.plan(counts)
            xp = be.pack_groups(x, slots, slots.shape[1], counts, offsets, T, T)
            be.grouped_gemm(xp, self.w1, counts, offsets, tiles, h, act=1)
        else:
            offsets, tiles, _ = be.plan(counts)
            be.grouped_gemm(x, self.w1, counts, offsets, tiles, h, row_src=slots, src_stride=slots.shape[1], act=1)
        out = torch.empty((T, self.d_model), dtype=x.dtype, device=x.device)
        be.grouped_gemm(h, self.w2, counts, offsets, tiles, out, row_dst=slots, dst_stride=slots.shape[1],
                        row_scale=gate)
        self.stats = MoEStats(tokens=T, sent=0, received=T)
        return out

    def _forward_ep(self, x, logits):
        import torch.distributed as dist

        torch = self._torch
        be = self.backend
        W, El, E = self.world, self.El, self.E
        T = x.shape[0]
        expert, gate, counts, slots = be.route(logits)
        offsets, _, perm = be.plan(counts, slots, slots.shape[1], T)
        send = be.gather_rows(x, perm, T)  # SRead: tokens in expert (= destination rank) order
        recv_counts = torch.empty(W * El, dtype=torch.int32, device=counts.device)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        # split sizes are host-side arguments of all-to-all-v: one small D2H for both directions
        both = torch.cat([offsets[::El], recv_counts.view(W, El).sum(dim=1, dtype=torch.int32)]).cpu().tolist()
        send_off = both[: W + 1]
        send_splits = [send_off[r + 1] - send_off[r] for r in range(W)]
        recv_splits = both[W + 1 :]
        R = sum(recv_splits)
        recv = torch.empty((R, self.d_model), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(recv, send, recv_splits, send_splits, group=self.group)
        rows, lcounts = be.recv_plan(recv_counts.view(W, El), R)
        loff, ltiles, _ = be.plan(lcounts)
        h = torch.empty((R, self.d_ff), dtype=x.dtype, device=x.device)
        y = torch.empty((R, self.d_model), dtype=x.dtype, device=x.device)
        if R:
            be.grouped_gemm(recv, self.w1, lcounts, loff, ltiles, h, row_src=rows, src_stride=rows.shape[1], act=1)
            be.grouped_gemm(h, self.w2, lcounts, loff, ltiles, y, row_dst=rows, dst_stride=rows.shape[1])
        back = torch.empty((T, self.d_model), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(back, y, send_splits, recv_splits, group=self.group)
        out = torch.empty((T, self.d_model), dtype=x.dtype, device=x.device)
        be.scatter_rows_scaled(back, perm, T, gate, out)  # SWrite * gate back to token order
        self.stats = MoEStats(tokens=T, sent=T, received=R)
        return out


def switch_flops(tokens: int, d_model: int, d_ff: int) -> float:
    """Expert FFN FLOPs of a top-1 layer: two GEMMs per token."""
    return 4.0 * tokens * d_model * d_ff
