#!/usr/bin/env python
"""PIT hot-path benchmark on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

A step is one pass of the PIT hot path over one synthetic batch: online detection of the
sparse operand's live micro-tiles from its values (K1, ``build_index_from_tensor``) followed by
the PIT sparse matmul against that index (``run_matmul_with_index``). The headline workload is
BASELINE config C1's distribution — random 32x1 micro-tiles, 90% zero, PIT axis k — at the
roofline scale SURVEY.md section 8(d) names (8192^3, bf16; C1's 1024^3 fp32 is the parity and
CPU-comparison size and is covered by the tests).

metric  = effective TFLOP/s: 2 * N * (A elements inside live micro-tiles) per step / step time
value   = device-resident inputs, CUDA events on the launching stream, L2 flushed between steps
e2e     = same metric through the public API with host (pinned) buffers, H2D + D2H inside the timing
roofline= the dominant kernel (spmm_gk) vs the measured bf16 peak (MEASURED_PEAKS.json)
--impl reference = the reference algorithm's CPU restatement (oracle/, the reference itself is
          pure Python and cannot travel) on the host cores, bounded sample of the same workload.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # the reference is fastest single-threaded

import argparse
import json
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: geometry of the sparse matmul C[M,N] = A[M,K] @ B[K,N]
    "pitk_c1_8192": dict(M=8192, K=8192, N=8192, micro=(32, 1), axis="k", zero=0.90, tile=(32, 64, 32),
                         desc="pit:k SpMM, C1 distribution (random 32x1 micro-tiles, 90% zero) at 8192^3 bf16; "
                              "online detection from values + SpMM"),
    "pitk_128_8192": dict(M=8192, K=8192, N=8192, micro=(128, 1), axis="k", zero=0.90, tile=(128, 64, 256),
                          desc="pit:k SpMM, B200-native 128x1 micro-tiles, 90% zero, 8192^3 bf16"),
    "pitk_256_8192": dict(M=8192, K=8192, N=8192, micro=(256, 1), axis="k", zero=0.90, tile=(256, 64, 256),
                          desc="pit:k SpMM, B200-native 256x1 micro-tiles on CTA pairs, 90% zero, 8192^3 bf16"),
    "pitm_32_8192": dict(M=8192, K=8192, N=8192, micro=(1, 32), axis="m", zero=0.90, tile=(16, 32, 128),
                         desc="pit:m SpMM, random 1x32 micro-tiles, 90% zero, 8192^3 bf16"),
    "bert_ffn1": dict(M=4096, K=768, N=3072, micro=(1, 768), axis="m", zero=None, tile=(128, 768, 256),
                      desc="BERT-base FFN1 varlen (batch 32 x 128, lengths U[16,128]), padding removed via pit:m"),
}
DEFAULT_WORKLOAD = "pitk_c1_8192"
# BASELINE configs[0] itself: the reference's CPU case (fp32, TF32 off) -- the `c1_fp32_1024` section
C1_1024 = dict(M=1024, K=1024, N=1024, micro=(32, 1), axis="k", zero=0.90, tile=(32, 64, 32),
               desc="BASELINE configs[0]: pit:k SpMM 1024^3 fp32, random 32x1 micro-tiles, 90% zero")
FLUSH_BYTES = 256 << 20
# CUDA event timestamps come in ~2 us quanta on this part (a 1-kernel graph replay reads 6.1 / 8.2 us,
# nothing between): per-replay times are averaged (mean), which resolves below the quantum, rather
# than taking a median that sits on the grid
L2_GATHER_PROBE_GBPS = 11145.6  # best L2->SM cp.async gather rate of the r1 probe (profiles/r1/copy_probe_l2_patterns.txt)
LTS_BYTES_PER_CYCLE = 6300  # whole-chip L2 (LTS) throughput cap, B300 notes (B300_MICROARCH.md, "LTS throughput cap")


# ------------------------------------------------------------------------------- bench CSV
# `pittile bench --csv` columns (reference cli.py:330) followed by the B200 roofline columns
CSV_COLUMNS = ["op", "shape", "granularity", "zero_ratio", "plan", "microtile", "tile", "launches", "wall_ms",
               "dense_wall_ms", "speedup", "eff_tflops", "gbps", "roofline_frac"]


def write_bench_csv(path, rows) -> None:
    """rows: dicts keyed by CSV_COLUMNS (values already formatted like the reference's: ms to 3
    decimals, speedup to 3)."""
    lines = [",".join(CSV_COLUMNS)] + [",".join(str(r.get(c, "")) for c in CSV_COLUMNS) for r in rows]
    Path(path).write_text("\n".join(lines) + "\n")


def read_bench_csv(path):
    """Rows of a `pittile bench` CSV or of ours (extra columns are kept when present)."""
    lines = Path(path).read_text().splitlines()
    head = lines[0].split(",")
    return [dict(zip(head, ln.split(","))) for ln in lines[1:] if ln.strip()]


# ----------------------------------------------------------------------------------- helpers
def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=float(d["hbm_gbs"]), bf16=float(d["bf16_tflops"]),
                    bf16_sustained=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), source="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sustained=1400.0, source="fallback")


def load_traffic():
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return {}
    return {}


class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def max_over_ranks(v: float, dev) -> float:
    """Max of a per-rank float over all ranks (NCCL on the device; a gloo rehearsal group on the host)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------------- synthetic inputs
def make_operands(w: dict, seed: int, device):
    """Synthetic A (sparse, masked at micro-tile granularity), B dense; bf16 on `device`."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    M, K, N = w["M"], w["K"], w["N"]
    t0, t1 = w["micro"]
    if w["name"].startswith("bert"):
        rng = np.random.default_rng(seed)
        lengths = rng.integers(16, 129, size=M // 128)
        rows = torch.from_numpy(np.concatenate([np.arange(128) < L for L in lengths])).to(device)
        A = torch.randn((M, K), device=device, dtype=torch.bfloat16, generator=g) * rows[:, None].to(torch.bfloat16)
        live_elems = int(rows.sum().item()) * K
    elif w["axis"] == "k":
        # A column-major: build A^T [K, M] row-major; micro-tile (t0, 1) = t0 consecutive m of one k
        keep = torch.rand((K, -(-M // t0)), device=device, generator=g) >= w["zero"]
        At = torch.randn((K, M), device=device, dtype=torch.bfloat16, generator=g)
        At.mul_(keep.repeat_interleave(t0, dim=1)[:, :M].to(torch.bfloat16))
        A = At.t()
        live_elems = int(keep.sum().item()) * t0
    else:
        keep = torch.rand((M, -(-K // t1)), device=device, generator=g) >= w["zero"]
        A = torch.randn((M, K), device=device, dtype=torch.bfloat16, generator=g)
        A.mul_(keep.repeat_interleave(t1, dim=1)[:, :K].to(torch.bfloat16))
        live_elems = int(keep.sum().item()) * t1
    B = torch.randn((K, N), device=device, dtype=torch.bfloat16, generator=g)
    return A, B, live_elems


def make_plan(w: dict):
    import paper_2301_10936_b200 as pit

    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    if reg.get("matmul", w["tile"]) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tuple(w["tile"]), "bench"))
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=w["M"], k=w["K"], n=w["N"]))
    plan = pit.forced_plan(expr, w["axis"], reg, tile_shape=w["tile"])
    assert tuple(plan.micro_tile) == tuple(w["micro"]), (plan.micro_tile, w["micro"])
    return plan


# --------------------------------------------------------------------------- our arm (GPU)
def run_ours(args, w):
    import torch
    import torch.distributed as dist

    import paper_2301_10936_b200 as pit
    from paper_2301_10936_b200 import _lib

    rank, world, local = dist_env()
    # PIT_BENCH_PG=gloo PIT_BENCH_DEVICE=0: rehearsal of the N-rank path with every rank on one GPU
    # (functional check of the multi-rank code on a 1-GPU box; its timings are not scaling numbers)
    if os.environ.get("PIT_BENCH_DEVICE") is not None:
        local = int(os.environ["PIT_BENCH_DEVICE"])
    if world > 1:
        if os.environ.get("PIT_BENCH_PG", "nccl") == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _lib.load()

    A, B, live = make_operands(w, seed=1234 + rank, device=dev)
    eff_flops = 2.0 * w["N"] * live
    plan = make_plan(w)
    micro, axis = w["micro"], w["axis"]
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        idx = pit.build_index_from_tensor(A, micro, axis)
        mark = torch.cuda.Event(enable_timing=True)
        mark.record(stream)
        C = pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx)
        return C, idx, mark

    # correctness spot check of the benchmarked configuration (cheap, outside timing)
    C0, idx0, _ = step()
    assert idx0.total * micro[0] * micro[1] >= live or w["name"].startswith("bert")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # kernel-level split (detection vs SpMM) measured through the eager API
    det_ms, spmm_ms = [], []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, _, e1 = step()
        e2.record(stream)
        det_ms.append((e0, e1))
        spmm_ms.append((e1, e2))
    torch.cuda.synchronize()
    det_ms = [a.elapsed_time(b) for a, b in det_ms]
    spmm_ms = [a.elapsed_time(b) for a, b in spmm_ms]
    # detection alone on the device (scan + compaction captured in a CUDA graph: no host dispatch
    # between the two launches), L2 flushed before each replay
    det_dev_ms = None
    try:
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            pit.build_index_from_tensor(A, micro, axis)
        stream.wait_stream(side)
        torch.cuda.synchronize()
        g_det = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_det):
            pit.build_index_from_tensor(A, micro, axis)
        for _ in range(3):
            g_det.replay()
        ev = []
        for _ in range(args.steps):
            flush.zero_()
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            g_det.replay()
            d1.record(stream)
            ev.append((d0, d1))
        torch.cuda.synchronize()
        det_dev_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
        del g_det
    except Exception:  # graph capture is an optimisation of the measurement, never a failure
        det_dev_ms = None
    # the step as a served layer runs it: detection + SpMM captured once in a CUDA graph, replayed
    captured = None
    if not args.no_graph:
        from paper_2301_10936_b200.graph import CapturedSparseMatmul

        captured = CapturedSparseMatmul(plan, A, B)
        for _ in range(args.warmup):
            captured.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    launches0 = _lib.kernel_launches()
    step_ev = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if captured is not None:
                captured.replay()
            else:
                step()
            e1.record(stream)
            step_ev.append((e0, e1))
        torch.cuda.synchronize()
    launches = (captured.kernels_per_replay * args.steps) if captured is not None else \
        (_lib.kernel_launches() - launches0)
    # the timed replays must compute what the eager public calls compute (deterministic kernels)
    replay_ok = bool(torch.equal(captured.C, C0.array)) if captured is not None else None
    total_ms = sum(a.elapsed_time(b) for a, b in step_ev)
    if world > 1:
        total_ms = max_over_ranks(total_ms, dev)
        dist.barrier()
    ms_per_step = total_ms / args.steps
    value = world * eff_flops * args.steps / (total_ms * 1e-3) / 1e12

    peaks = load_peaks()
    spmm_avg = statistics.mean(spmm_ms)
    det_avg = statistics.mean(det_ms)
    achieved = eff_flops / (spmm_avg * 1e-3) / 1e12
    scanned = A.numel() * A.element_size()
    traffic = load_traffic().get(w["name"], {}).get("spmm_dram_bytes")
    operand_feed = None
    if axis == "k":
        # gathered operand bytes per launch: every live (group, k) pair brings one B row strip of
        # the n tile and one A^T strip of the group, for every n tile (csrc/pit_spmm_tc.cu spmm_gk)
        gw = micro[0]
        pair = gw > 128 and w["N"] > 128 and os.environ.get("PIT_GK2", "1") != "0"  # spmm_gk2 (CTA pairs)
        n_tile = 256 if (gw < 256 or pair) else 128
        if gw <= 32 and w["N"] >= 1024 and os.environ.get("PIT_GK_NT") not in ("128", "256"):
            n_tile = 512  # 16/32-row groups over wide N: 512-column units (csrc dispatch_tc)
        gathered = idx0.total * (-(-w["N"] // n_tile)) * (n_tile + gw) * 2
        feed = gathered / (spmm_avg * 1e-3) / 1e9
        lts_cap = LTS_BYTES_PER_CYCLE * (clocks.summary().get("sm_mhz") or 1965.0) * 1e6 / 1e9
        operand_feed = {"bytes_per_launch": gathered, "achieved_GBps": round(feed, 1),
                        "ceiling_GBps": round(lts_cap, 1), "frac": round(feed / lts_cap, 4),
                        "ceiling_source": "L2 (LTS) throughput cap ~6300 B/cycle x the measured SM clock (B300 notes; "
                                          "the gathered operands stream from L2)",
                        "r1_probe_GBps": L2_GATHER_PROBE_GBPS}
    roofline = {
        "bound": "tensor", "kernel": ("spmm_gk2" if axis == "k" and micro[0] > 128 and w["N"] > 128 and os.environ.get("PIT_GK2", "1") != "0" else "spmm_gk") if axis == "k" else "spmm_gm",
        "achieved": round(achieved, 2), "peak": peaks["bf16"], "unit": "TFLOP/s",
        "frac": round(achieved / peaks["bf16"], 4), "peak_source": peaks["source"] + " burst bf16",
        "traffic": traffic, "algorithmic_flops": eff_flops,
        "kernel_ms": round(spmm_avg, 4), "operand_feed": operand_feed,
    }
    det_t = det_dev_ms if det_dev_ms else det_avg
    detection = {
        "kernel": "detect+compact (" + ("CUDA graph of the public call, device time" if det_dev_ms else
                                       "eager call incl. host dispatch") + ")",
        "ms": round(det_t, 4), "bytes_scanned": scanned,
        "achieved_GBps": round(scanned / (det_t * 1e-3) / 1e9, 1), "peak_GBps": peaks["hbm"],
        "frac": round(scanned / (det_t * 1e-3) / 1e9 / peaks["hbm"], 4),
        "eager_ms_incl_host_dispatch": round(det_avg, 4),
    }

    result = {
        "metric": "PIT sparse matmul effective TFLOP/s (online detection + SpMM)",
        "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": base_config(w, world),
        "execution": "CUDA graph of detect+SpMM (paper_2301_10936_b200.graph)" if not args.no_graph
                     else "eager API calls",
        "roofline": roofline, "detection": detection,
        "clocks": clocks.summary(), "gpu_launches": int(launches),
        "graph_replay_equals_eager": replay_ok,
    }

    if world > 1:
        # N > 1: the single-operator sections are per-GPU replicas of the N=1 numbers (north_star reports
        # them at 1 GPU); only the headline replica step and the expert-parallel MoE layer run
        args.no_index_bench = args.no_sweep = args.no_bert = args.no_attn = args.no_opt = True
    if not args.no_index_bench:
        result["index_build"] = index_build_bench(dev, peaks)
    if not args.no_sweep:
        try:
            result["sparsity_sweep"] = sparsity_sweep_bench(args, dev, peaks)
        except Exception as e:
            result["sparsity_sweep"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if not args.no_bert and w["name"] != "bert_ffn1":
        try:
            result["bert_ffn1"] = bert_bench(args, dev, peaks)
        except Exception as e:
            result["bert_ffn1"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if not args.no_attn:
        try:
            result["attention"] = attention_bench(args, dev, peaks)
        except Exception as e:
            result["attention"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if not args.no_opt:
        try:
            result["opt_ffn2"] = opt_bench(args, dev, peaks)
        except Exception as e:
            result["opt_ffn2"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if not args.no_moe:
        try:
            result["moe"] = moe_bench(args, world, rank, dev, peaks)
        except Exception as e:  # never lose the headline line to the secondary workload
            result["moe"] = {"error": f"{type(e).__name__}: {e}"[:300]}

    # ---- end to end through the public API with host buffers
    if rank == 0 and not args.no_e2e:
        result["e2e"] = e2e_ours(args, w, A, B, plan, eff_flops)
    if rank == 0 and not args.no_c1 and world == 1:
        try:
            result["c1_fp32_1024"] = c1_fp32_bench(args, dev, peaks)
        except Exception as e:
            result["c1_fp32_1024"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        # the reference's CPU path beside every section (1 core and all host cores, CPU model stated)
        names = [w["name"]] + [s for s, key in (("c1_1024", "c1_fp32_1024"), ("bert_ffn1", "bert_ffn1"),
                                                  ("attention", "attention"), ("opt_ffn2", "opt_ffn2"),
                                                  ("moe", "moe")) if isinstance(result.get(key), dict)
                                and "error" not in result[key]]
        cpu = cpu_sections_subprocess(names, args.cpu_seconds)
        result["cpu_baseline"] = cpu.pop(w["name"], {"error": "missing"})
        for s, key in (("c1_1024", "c1_fp32_1024"), ("bert_ffn1", "bert_ffn1"), ("attention", "attention"),
                       ("opt_ffn2", "opt_ffn2"), ("moe", "moe")):
            if s in cpu:
                result[key]["cpu_baseline"] = cpu[s]
    if world > 1:
        dist.destroy_process_group()
    return result if rank == 0 else None


def pit_run(plan, A, B, w):
    """The eager public calls of one step (reference output for a captured graph)."""
    import paper_2301_10936_b200 as pit

    idx = pit.build_index_from_tensor(A, w["micro"], w["axis"])
    return pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx).array


def _graph_ms(fn, flush, reps):
    """Mean device time of fn() captured in a CUDA graph, L2 flushed before each replay (event
    timestamps come in ~2 us quanta, so the mean, not the median, resolves below that)."""
    import torch

    stream = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    stream.wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        fn()
    for _ in range(3):
        graph.replay()
    ev = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        graph.replay()
        e1.record(stream)
        ev.append((e0, e1))
    torch.cuda.synchronize()
    del graph
    return statistics.mean(a.elapsed_time(b) for a, b in ev)


def bert_bench(args, dev, peaks):
    """C2 (BASELINE configs[1]): BERT-base FFN1 over a variable-length batch (32 sequences of
    U[16,128] tokens padded to 128), padding removed via pit:m with row-uniform (1, 768) micro-tiles:
    online detection from the activations + the gathered-row GEMM, one CUDA graph, L2 flushed.
    Effective FLOPs = 2 * 3072 * live elements (padding excluded)."""
    import torch

    import paper_2301_10936_b200 as pit
    from paper_2301_10936_b200.graph import CapturedSparseMatmul

    w = dict(WORKLOADS["bert_ffn1"], name="bert_ffn1")
    A, B, live = make_operands(w, seed=1234, device=dev)  # the --workload bert_ffn1 operands
    eff = 2.0 * w["N"] * live
    plan = make_plan(w)
    eager = pit_run(plan, A, B, w)
    captured = CapturedSparseMatmul(plan, A, B)
    for _ in range(max(3, args.warmup)):
        captured.replay()
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    ev = []
    for _ in range(max(5, args.steps)):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        captured.replay()
        e1.record(stream)
        ev.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    # context on the same box: the same product dense on the padded batch (cuBLAS and this package's
    # dense plan), cuBLAS on the live rows alone (the floor for any padding removal), and the pit:m
    # product with the index reused (what each further layer of a batch pays: PIT builds one index
    # per batch)
    rows = int(live // w["K"])
    Al = torch.randn((rows, w["K"]), device=dev, dtype=torch.bfloat16)
    row_live = (A != 0).any(dim=1).cpu().numpy()  # the token rows the sequence lengths keep
    ann_rows = pit.from_bits(row_live[:, None], (w["M"], w["K"]), (1, w["K"])).on_device(dev)
    ctx_reps = max(20, args.steps)
    idx = pit.build_index_from_tensor(A, w["micro"], w["axis"])
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    dplan = pit.forced_plan(pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"),
                                             dict(m=w["M"], k=w["K"], n=w["N"])), "dense", reg, tile_shape=(128, 64, 256))
    context = {
        "cublas_padded_ms": round(_graph_ms(lambda: torch.matmul(A, B), flush, ctx_reps), 4),
        "cublas_live_rows_ms": round(_graph_ms(lambda: torch.matmul(Al, B), flush, ctx_reps), 4),
        "pit_dense_padded_ms": round(_graph_ms(lambda: pit.run_matmul_with_index(
            dplan, pit.DenseTensor(A), pit.DenseTensor(B), None), flush, ctx_reps), 4),
        "pit_m_index_reused_ms": round(_graph_ms(lambda: pit.run_matmul_with_index(
            plan, pit.DenseTensor(A), pit.DenseTensor(B), idx), flush, ctx_reps), 4),
        # the padding known from the sequence lengths instead of detected from the values: the
        # annotation (1 bit per token row) on the device, index built from its bits
        "pit_m_from_lengths_ms": round(_graph_ms(lambda: pit.run_matmul_with_index(
            plan, pit.DenseTensor(A), pit.DenseTensor(B), pit.build_index(ann_rows, w["micro"], w["axis"])),
            flush, ctx_reps), 4),
        "timing": "mean of CUDA-graph replays, L2 flushed before each",
    }
    return {"workload": w["desc"], "value": round(eff / (ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s (effective)",
            "ms_per_step": round(ms, 4), "step_mean_ms": round(statistics.mean(a.elapsed_time(b) for a, b in ev), 4),
            "live_rows": rows, "rows": w["M"], "context": context,
            "frac_bf16_peak": round(eff / (ms * 1e-3) / 1e12 / peaks["bf16"], 4),
            "graph_replay_equals_eager": bool(torch.equal(captured.C, eager)),
            "execution": "CUDA graph: build_index_from_tensor (1, 768) + run_matmul_with_index (pit:m)"}


def _time_layer(fn, steps, dev, world):
    """Mean per-call device time of fn() (CUDA events on the current stream), max over ranks."""
    import torch
    import torch.distributed as dist

    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        ev.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        ms = max_over_ranks(ms, dev)
    return ms


def moe_bench(args, world, rank, dev, peaks, tokens_per_gpu=16384, n_experts=128, d_model=768, d_ff=3072):
    """C5: Switch-base-128 MoE layer (top-1, dropless), tokens sharded per GPU (weak scaling), experts
    sharded over ranks (expert parallelism) when world > 1. Synthetic activations, Gaussian router
    logits (imbalanced top-1), random bf16 expert weights. Layer time = route + index + dispatch +
    FFN1(ReLU) + FFN2 + combine (router GEMM excluded), one CUDA graph per layer, max over ranks.
    world > 1: the product exchange is the peer-memory one (csrc/pit_ep.cu: dispatch stores token rows
    into the expert rank's region over NVLink, combine pulls them back, no host sync); the NCCL
    all-to-all-v orchestration is timed beside it as the baseline (eager: it needs a D2H of the
    split sizes)."""
    import torch
    import torch.distributed as dist

    from paper_2301_10936_b200 import _lib
    from paper_2301_10936_b200.moe import SwitchMoE, switch_flops

    E, El = n_experts, n_experts // world
    g = torch.Generator(device=dev).manual_seed(7 + rank)
    x = torch.randn((tokens_per_gpu, d_model), device=dev, dtype=torch.bfloat16, generator=g)
    logits = torch.randn((tokens_per_gpu, E), device=dev, dtype=torch.float32, generator=g)
    w1 = (torch.randn((El, d_model, d_ff), device=dev, generator=g) / d_model ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn((El, d_ff, d_model), device=dev, generator=g) / d_ff ** 0.5).to(torch.bfloat16)
    group = dist.group.WORLD if world > 1 else None
    layer = SwitchMoE(w1, w2, E, group=group, capacity=tokens_per_gpu)
    steps = max(5, args.steps)
    for _ in range(max(3, args.warmup)):
        eager = layer(x, logits)
    torch.cuda.synchronize()
    graphable = layer.exchange != "nccl"  # the all-to-all-v fallback reads split sizes on the host
    if world > 1:
        dist.barrier()
    if graphable:
        # the layer as a served model runs it: one CUDA graph (no host round trip on either path)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            layer(x, logits)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        graph = torch.cuda.CUDAGraph()
        launches0 = _lib.kernel_launches()
        with torch.cuda.graph(graph):
            out_g = layer(x, logits)
        launches_per_layer = _lib.kernel_launches() - launches0
        for _ in range(max(3, args.warmup)):
            graph.replay()
        ms = _time_layer(graph.replay, steps, dev, world)
        replay_ok = bool(torch.equal(out_g, eager))
    else:
        launches0 = _lib.kernel_launches()
        layer(x, logits)
        launches_per_layer = _lib.kernel_launches() - launches0
        ms = _time_layer(lambda: layer(x, logits), steps, dev, world)
        replay_ok = None
    ep_error = layer._peer.error() if layer._peer is not None else 0
    baseline = None
    if world > 1 and dist.get_backend() == "nccl":
        nccl = SwitchMoE(w1, w2, E, group=group, exchange="nccl")
        for _ in range(max(3, args.warmup)):
            ref_out = nccl(x, logits)
        nccl_ms = _time_layer(lambda: nccl(x, logits), steps, dev, world)
        same = bool(torch.equal(ref_out, eager))
        baseline = {"exchange": "NCCL all_to_all_single (counts) + D2H of split sizes + all-to-all-v x2, eager",
                    "ms_per_layer": round(nccl_ms, 4),
                    "tokens_per_s": round(world * tokens_per_gpu / (nccl_ms * 1e-3), 1),
                    "output_equals_peer_path": same}
    received = int(layer._peer.lcounts.sum().item()) if layer._peer is not None else tokens_per_gpu
    peer_self = None
    if world == 1:
        # the peer-memory exchange kernels against this rank's own region (dispatch stores + combine
        # pulls through the region instead of the fused gather / scaled-scatter GEMM epilogues)
        selfx = SwitchMoE(w1, w2, E, exchange="peer", capacity=tokens_per_gpu)
        for _ in range(max(3, args.warmup)):
            so = selfx(x, logits)
        ps_ms = _time_layer(lambda: selfx(x, logits), steps, dev, world)
        peer_self = {"ms_per_layer": round(ps_ms, 4), "tokens_per_s": round(tokens_per_gpu / (ps_ms * 1e-3), 1),
                     "max_abs_diff_vs_local": float((so.float() - eager.float()).abs().max()),
                     "timeouts": selfx._peer.error(), "execution": "eager"}
        selfx.close()
    if world > 1:
        layer.close()
        dist.barrier()
    toks = world * tokens_per_gpu / (ms * 1e-3)
    flops = switch_flops(world * tokens_per_gpu, d_model, d_ff) / (ms * 1e-3) / 1e12
    # HBM roofline of one rank's layer: its experts' weights are streamed once (2 matrices x El x
    # d_model x d_ff bf16) plus the token rows read / written (x, hidden, output; exchange buffers
    # not counted). At 128 tokens per expert this, not the tensor pipe, bounds the layer.
    hbm_bytes = 2 * El * d_model * d_ff * 2 + received * (d_model * 2 * 2 + d_ff * 2 * 2) + tokens_per_gpu * d_model * 2 * 2
    hbm_gbps = hbm_bytes / (ms * 1e-3) / 1e9
    out = {"metric": "MoE layer tokens/s", "value": round(toks, 1), "unit": "tokens/s", "n_gpus": world,
           "ms_per_layer": round(ms, 4), "expert_tflops_per_gpu": round(flops / world, 2),
           "frac_bf16_peak": round(flops / world / peaks["bf16"], 4),
           "roofline": {"bound": "hbm", "achieved": round(hbm_gbps, 1), "peak": peaks["hbm"], "unit": "GB/s",
                        "frac": round(hbm_gbps / peaks["hbm"], 4), "traffic": None,
                        "algorithmic_bytes_per_layer": int(hbm_bytes),
                        "note": "expert weights streamed once per layer dominate; tensor-time floor "
                                f"{switch_flops(tokens_per_gpu, d_model, d_ff) / peaks['bf16'] / 1e9:.3f} ms vs HBM floor "
                                f"{hbm_bytes / peaks['hbm'] / 1e6:.3f} ms"},
           "config": {"experts": E, "experts_per_gpu": El, "d_model": d_model, "d_ff": d_ff,
                      "tokens_per_gpu": tokens_per_gpu, "routing": "top-1 argmax, Gaussian logits, dropless",
                      "parallelism": f"ep{world}" if world > 1 else "single GPU", "received_rank0": received,
                      "exchange": layer.exchange, "peer_fallback": layer.fallback_reason,
                      "execution": "CUDA graph of the whole layer" if graphable else "eager (all-to-all-v fallback)"},
           "gpu_launches_per_layer": int(launches_per_layer), "graph_replay_equals_eager": replay_ok,
           "exchange_timeouts": int(ep_error)}
    if world > 1:
        # the exchange's own floor: every rank sends and receives its tokens twice over NVLink
        xbytes = 2 * tokens_per_gpu * d_model * 2
        out["exchange"] = {"bytes_per_rank_per_layer": xbytes, "nvlink_floor_ms": round(xbytes / 900e9 * 1e3, 4)}
        out["baseline_nccl"] = baseline
    else:
        out["peer_exchange_one_rank"] = peer_self
    return out


def sparsity_sweep_bench(args, dev, peaks, side=8192, micros=((32, 1), (128, 1), (256, 1)),
                         zeros=(0.5, 0.9, 0.95, 0.99), reps=5):
    """"Effective TFLOP/s vs sparsity" (BASELINE metric) for the pit:k product at 8192^3 bf16: every
    micro-tile height the tcgen05 kernels tile natively (32x1 = C1's, 128x1, 256x1 on CTA pairs),
    random micro-tile sparsity 50..99%. SpMM kernel time alone (CUDA events on the launching stream,
    L2 flushed before each call; the index is built once per configuration, outside the timing),
    and the index build from values (detect + compaction) beside it."""
    import torch

    import paper_2301_10936_b200 as pit

    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    out = {}
    for micro in micros:
        for zero in zeros:
            w = dict(M=side, K=side, N=side, micro=micro, axis="k", zero=zero, tile=(micro[0], 64, 256),
                     name=f"sweep_{micro[0]}x{micro[1]}_{zero}")
            A, B, live = make_operands(w, seed=99, device=dev)
            plan = make_plan(w)
            flops = 2.0 * side * live
            idx = pit.build_index_from_tensor(A, micro, "k")
            for _ in range(2):
                pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx)
            ev = []
            for _ in range(reps):
                flush.zero_()
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record(stream)
                idx = pit.build_index_from_tensor(A, micro, "k")
                e1.record(stream)
                pit.run_matmul_with_index(plan, pit.DenseTensor(A), pit.DenseTensor(B), idx)
                e2.record(stream)
                ev.append((e0, e1, e2))
            torch.cuda.synchronize()
            det = statistics.mean(a.elapsed_time(b) for a, b, _ in ev)
            mm = statistics.mean(b.elapsed_time(c) for _, b, c in ev)
            tf = flops / (mm * 1e-3) / 1e12
            kern = "spmm_gk2 (CTA pair)" if micro[0] > 128 else "spmm_gk"
            out[f"{micro[0]}x{micro[1]}@{zero}"] = {
                "kernel": kern, "spmm_ms": round(mm, 4), "effective_TFLOPs": round(tf, 1),
                "frac_bf16_peak": round(tf / peaks["bf16"], 4), "live_fraction": round(live / side / side, 4),
                "index_build_ms": round(det, 4),
                "index_build_GBps": round(A.numel() * 2 / (det * 1e-3) / 1e9, 1)}
            del A, B, idx
    return {"workload": f"pit:k SpMM {side}^3 bf16, random micro-tile sparsity, online index from values",
            "peak_TFLOPs": peaks["bf16"], "by_microtile_and_zero_ratio": out}


def index_build_bench(dev, peaks, side=16384, reps=20):
    """K1 alone at the north-star size: online detection over a 16384^2 bf16 tensor (512 MiB),
    C1 distribution (32x1 micro-tiles, 90% zero, column-major like the pit:k operand), launches
    back to back so host overhead hides behind GPU time. Algorithmic bytes = tensor bytes + index
    bytes written."""
    import torch

    import paper_2301_10936_b200 as pit

    g = torch.Generator(device=dev).manual_seed(99)
    keep = torch.rand((side, side // 32), device=dev, generator=g) >= 0.9
    At = torch.randn((side, side), device=dev, dtype=torch.bfloat16, generator=g)
    At.mul_(keep.repeat_interleave(32, dim=1).to(torch.bfloat16))
    A = At.t()
    del keep
    idx = pit.build_index_from_tensor(A, (32, 1), "k")
    total = idx.total
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    times = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pit.build_index_from_tensor(A, (32, 1), "k")
        e1.record(stream)
        times.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in times)
    nbytes = A.numel() * 2 + 4 * (idx.n_groups + total)
    gbps = nbytes / (ms * 1e-3) / 1e9
    del At, A
    return {"workload": f"build_index_from_tensor, {side}x{side} bf16 column-major, micro (32,1), 90% zero",
            "ms": round(ms, 4), "bytes": nbytes, "achieved_GBps": round(gbps, 1), "peak_GBps": peaks["hbm"],
            "frac": round(gbps / peaks["hbm"], 4), "bound": "hbm", "l2": "flushed before each call"}


def longformer_blocks(heads, seq, rng, window=256, rand=0.02):
    """C3 block mask on the (32 query x 64 key) grid: sliding window +-`window`, the first key block
    global (every query sees it), the first query block global (sees every key), plus seeded random
    blocks. Returns bool [heads, seq/32, seq/64]."""
    qi = np.arange(seq // 32)[:, None] * 32 + 16
    kj = np.arange(seq // 64)[None, :] * 64 + 32
    base = np.abs(qi - kj) <= window + 48
    base[:, 0] = True
    base[0, :] = True
    return np.stack([base | (rng.random(base.shape) < rand) for _ in range(heads)])


def attention_bench(args, dev, peaks, heads=12, seq=4096, hd=64):
    """C3: Longformer-style block-sparse attention output O = P.V per head (seq 4096, head dim 64,
    32x64 blocks), all heads in ONE batched launch (slices stacked along queries). Two PIT plans
    over the same mask, both timed:
      pit:m, micro (1,64) on row-major P: row tiles of 128 queries, K-blocks of 64 keys in which no
        query of the tile is live are skipped (block rows are 32 queries, so skipping is exact at
        the 4-block-row level);
      pit:k, micro (32,1) on column-major P (P^T stored): gathered keys per 32-query group.
    Step = index build from the device-resident block mask + batched SpMM, in a CUDA graph.
    Effective FLOPs = 2 * hd * live P elements."""
    import torch

    import paper_2301_10936_b200 as pit

    rng = np.random.default_rng(3)
    blocks = longformer_blocks(heads, seq, rng)
    ann_dev = pit.from_bits(blocks.reshape(heads * seq // 32, seq // 64), (heads * seq, seq), (32, 64)).on_device(dev)
    live = int(blocks.sum()) * 32 * 64
    eff = 2.0 * hd * live
    g = torch.Generator(device=dev).manual_seed(5)
    emask = torch.from_numpy(blocks).to(dev).repeat_interleave(32, 1).repeat_interleave(64, 2)  # [h, q, k]
    P = torch.randn((heads, seq, seq), device=dev, dtype=torch.bfloat16, generator=g)
    P.mul_(emask.to(torch.bfloat16))
    del emask
    V = torch.randn((heads, seq, hd), device=dev, dtype=torch.bfloat16, generator=g)
    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    expr = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=seq, k=seq, n=hd))
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    ref = P[0].double() @ V[0].double()

    def timed(step):
        O = step()
        err = float((O[0].double() - ref).abs().max() / ref.abs().max().clamp_min(1e-6))
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                step()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            O_g = step()
        for _ in range(args.warmup):
            graph.replay()
        ev = []
        for _ in range(max(args.steps, 5)):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            ev.append((e0, e1))
        torch.cuda.synchronize()
        ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
        return {"ms_per_step": round(ms, 4), "value": round(eff / (ms * 1e-3) / 1e12, 2),
                "max_rel_err_head0_vs_f64": err, "graph_replay_equals_eager": bool(torch.equal(O_g, O))}

    variants = {}
    plan_m = pit.forced_plan(expr, "m", reg, tile_shape=(128, 64, 256))
    A3m = P  # row-major slices stacked along queries
    variants["pit:m (1,64) row-major P"] = timed(
        lambda: pit.run_batched_matmul_with_index(plan_m, A3m, V, pit.build_index(ann_dev, (1, 64), "m")))
    plan_k = pit.forced_plan(expr, "k", reg, tile_shape=(32, 64, 32))
    A3k = pit.stack_slices(P, plan_k)  # P^T stored: [keys, heads*queries]
    del P
    variants["pit:k (32,1) column-major P"] = timed(
        lambda: pit.run_batched_matmul_with_index(plan_k, A3k, V, pit.build_index(ann_dev, (32, 1), "k")))
    # B200-native wider query groups: micro-tile (128,1) covers four 32-query block rows (the union of
    # their keys; Longformer windows of adjacent query blocks overlap), 4x the MMA width per key
    tile128 = (128, 64, 256)
    if reg.get("matmul", tile128) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile128, "attn128"))
    plan_k128 = pit.forced_plan(expr, "k", reg, tile_shape=tile128)
    variants["pit:k (128,1) column-major P"] = timed(
        lambda: pit.run_batched_matmul_with_index(plan_k128, A3k, V, pit.build_index(ann_dev, (128, 1), "k")))
    # two 32-query block rows per group: half the union waste of (128,1), half its MMA width
    tile64 = (64, 64, 256)
    if reg.get("matmul", tile64) is None:
        reg.register(pit.TileKernelDescriptor("matmul", tile64, "attn64"))
    plan_k64 = pit.forced_plan(expr, "k", reg, tile_shape=tile64)
    variants["pit:k (64,1) column-major P"] = timed(
        lambda: pit.run_batched_matmul_with_index(plan_k64, A3k, V, pit.build_index(ann_dev, (64, 1), "k")))
    # online detection from the P values instead of the mask (K1 over the stacked 402 MB operand)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pit.build_batched_index_from_tensor(A3k, (32, 1), "k")
    flush.zero_()
    e0.record(stream)
    pit.build_batched_index_from_tensor(A3k, (32, 1), "k")
    e1.record(stream)
    torch.cuda.synchronize()
    det_ms = e0.elapsed_time(e1)
    best = max(variants, key=lambda k: variants[k]["value"])
    scores = attention_scores_bench(args, dev, peaks, blocks, ann_dev, heads, seq, hd, flush)
    out = {"workload": f"Longformer-style P.V: {heads} heads, seq {seq}, head dim {hd}, 32x64 blocks "
                       f"(window +-256, global first block row/col, 2% random), one batched launch for all heads",
           "value": variants[best]["value"], "unit": "TFLOP/s (effective)", "plan": best,
           "ms_per_step": variants[best]["ms_per_step"], "variants": variants,
           "density": round(live / (heads * seq * seq), 4), "effective_flops": eff,
           "frac_bf16_peak": round(variants[best]["value"] / peaks["bf16"], 4),
           # head dim 64: every gathered P value feeds 64 MACs, so the product is bound by reading the
           # live P blocks (plus V once and C once), not by the tensor pipe
           "roofline": {"bound": "hbm", "unit": "GB/s", "peak": peaks["hbm"],
                        "algorithmic_bytes": live * 2 + 2 * heads * seq * hd * 2,
                        "achieved": round((live * 2 + 2 * heads * seq * hd * 2)
                                          / (variants[best]["ms_per_step"] * 1e-3) / 1e9, 1),
                        "frac": round((live * 2 + 2 * heads * seq * hd * 2)
                                      / (variants[best]["ms_per_step"] * 1e-3) / 1e9 / peaks["hbm"], 4),
                        "note": "whole step (index build from the block mask + SpMM) against live P + V + C bytes"},
           "detect_from_values_ms": round(det_ms, 4),
           "detect_from_values_GBps": round(heads * seq * seq * 2 / (det_ms * 1e-3) / 1e9, 1),
           "execution": "CUDA graph: build_index(mask bits on device) + batched SpMM",
           "scores_sddmm": scores}
    del A3k
    return out


def attention_scores_bench(args, dev, peaks, blocks, ann_dev, heads, seq, hd, flush):
    """C3 producer side: S = Q.K^T per head only inside the 32x64 block mask, all heads
    in one output-sparse launch (csrc/pit_sddmm.cu), as a CUDA graph of the public call (both output
    indexes built from the device mask + the SDDMM), L2 flushed. Roofline: HBM — algorithmic bytes =
    live S written + Q + K read once. Dense cuBLAS Q.K^T (torch.bmm, every score) beside it."""
    import torch

    from paper_2301_10936_b200.sddmm import run_batched_sddmm

    g = torch.Generator(device=dev).manual_seed(17)
    Q = torch.randn((heads, seq, hd), device=dev, dtype=torch.bfloat16, generator=g)
    Kt = torch.randn((heads, seq, hd), device=dev, dtype=torch.bfloat16, generator=g)
    S = torch.zeros((heads, seq, seq), device=dev, dtype=torch.bfloat16)
    live = int(blocks.sum()) * 32 * 64
    stream = torch.cuda.current_stream()

    def step():
        return run_batched_sddmm(Q, Kt.transpose(1, 2), ann_dev, out=S)

    step()
    torch.cuda.synchronize()
    m = torch.from_numpy(blocks[0]).to(dev).repeat_interleave(32, 0).repeat_interleave(64, 1)
    ref = Q[0].double() @ Kt[0].double().t()
    err = float((S[0].double()[m] - ref[m]).abs().max() / ref[m].abs().max())
    eager = S.clone()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        step()
    stream.wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()

    def timed(fn, reps):
        for _ in range(3):  # warm-up: the first eager cuBLAS call carries its one-time setup
            fn()
        ev = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            ev.append((e0, e1))
        torch.cuda.synchronize()
        return statistics.mean(a.elapsed_time(b) for a, b in ev)

    for _ in range(3):
        graph.replay()
    ms = timed(graph.replay, max(args.steps, 5))
    replay_ok = bool(torch.equal(S, eager))
    Sd = torch.empty((heads, seq, seq), device=dev, dtype=torch.bfloat16)
    dense_ms = timed(lambda: torch.bmm(Q, Kt.transpose(1, 2), out=Sd), max(args.steps, 5))
    del Sd
    nbytes = live * 2 + 2 * heads * seq * hd * 2
    gbps = nbytes / (ms * 1e-3) / 1e9
    return {"ms_per_step": round(ms, 4), "effective_TFLOPs": round(2.0 * hd * live / (ms * 1e-3) / 1e12, 2),
            "roofline": {"bound": "hbm", "achieved": round(gbps, 1), "peak": peaks["hbm"], "unit": "GB/s",
                         "frac": round(gbps / peaks["hbm"], 4), "algorithmic_bytes": nbytes,
                         "note": "live S written + Q, K read once; step includes both output indexes built from the device mask"},
            "dense_cublas_bmm_ms": round(dense_ms, 4), "speedup_vs_dense": round(dense_ms / ms, 2),
            "max_rel_err_head0_vs_f64": err, "graph_replay_equals_eager": replay_ok,
            "execution": "CUDA graph: output_indexes(mask bits on device) + run_batched_sddmm"}


def opt_bench(args, dev, peaks, tokens=4096, d_model=2048, d_ff=8192, zeros=(0.9, 0.99)):
    """C4: OPT-1.3B FFN2 under dynamic activation sparsity, one training step's two sparse products
    (1x32 micro-tiles on the ReLU activations H [tokens, d_ff], bf16):
      forward   Y  = H . W2        pit:m, micro (1,32) (live token rows per 32-neuron K-block)
      backward  dW2 = H^T . dY     pit:k, micro (32,1) on H^T — H^T column-major IS H row-major, and
                                   its index is the forward index transposed (one detection)
    Step = detection from H's values + both products (CUDA graph). Effective FLOPs = 2 * 2048 *
    live(H) per product."""
    import torch

    import paper_2301_10936_b200 as pit

    reg = pit.register_builtin_kernels(include_b200_tiles=True)
    fwd_e = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=tokens, k=d_ff, n=d_model))
    bwd_e = pit.bind_extents(pit.parse_expr("C[m,n] += A[m,k] * B[k,n]"), dict(m=d_ff, k=tokens, n=d_model))
    plan_f = pit.forced_plan(fwd_e, "m", reg, tile_shape=(16, 32, 128))
    plan_b = pit.forced_plan(bwd_e, "k", reg, tile_shape=(32, 64, 32))
    g = torch.Generator(device=dev).manual_seed(11)
    W2 = torch.randn((d_ff, d_model), device=dev, dtype=torch.bfloat16, generator=g) * 0.02
    dY = torch.randn((tokens, d_model), device=dev, dtype=torch.bfloat16, generator=g)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    out = {"workload": f"OPT-1.3B FFN2, {tokens} tokens (8x512), d_ff {d_ff} -> d_model {d_model}, ReLU activations "
                       "with random 1x32 micro-tile sparsity; fwd pit:m + weight-grad pit:k from one detection",
           "unit": "TFLOP/s (effective)", "by_zero_ratio": {}}
    for zr in zeros:
        keep = torch.rand((tokens, d_ff // 32), device=dev, generator=g) >= zr
        H = torch.relu(torch.randn((tokens, d_ff), device=dev, dtype=torch.bfloat16, generator=g))
        H.mul_(keep.repeat_interleave(32, dim=1).to(torch.bfloat16))
        live = int(keep.sum().item()) * 32
        eff = 2 * 2.0 * d_model * live

        def step():
            idx = pit.build_index_from_tensor(H, (1, 32), "m")
            Y = pit.run_matmul_with_index(plan_f, pit.DenseTensor(H), pit.DenseTensor(W2), idx)
            dW2 = pit.run_matmul_with_index(plan_b, pit.DenseTensor(H.t()), pit.DenseTensor(dY), idx.transposed())
            return Y.array, dW2.array

        Y, dW2 = step()
        ry = H.double() @ W2.double()
        rw = H.t().double() @ dY.double()
        err = max(float((Y.double() - ry).abs().max() / ry.abs().max()), float((dW2.double() - rw).abs().max() /
                                                                                 rw.abs().max()))
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                step()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            O_g = step()
        for _ in range(args.warmup):
            graph.replay()
        ev = []
        for _ in range(max(args.steps, 5)):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            ev.append((e0, e1))
        torch.cuda.synchronize()
        ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
        # per-product split: each product alone as a CUDA graph over the step's index, L2 flushed
        idx = pit.build_index_from_tensor(H, (1, 32), "m")
        split = []
        for plan, A, B, ix in ((plan_f, H, W2, idx), (plan_b, H.t(), dY, idx.transposed())):
            split.append(_graph_ms(lambda plan=plan, A=A, B=B, ix=ix: pit.run_matmul_with_index(
                plan, pit.DenseTensor(A), pit.DenseTensor(B), ix), flush, max(args.steps, 10)))
        # the rest of FFN2's backward: dH = (dY . W2^T) * 1[H > 0] only inside H's live 1x32
        # micro-tiles -- the output-sparse plan (SDDMM, K8) with the ReLU gate, annotation detected
        # from H on the device each step; dense cuBLAS dY . W2^T (every element) beside it
        from paper_2301_10936_b200.sddmm import run_sddmm_like

        dH = torch.zeros_like(H)

        def dh_step():
            run_sddmm_like(dY, W2.t(), H, (1, 32), out=dH, gate=H)

        dh_step()
        dh_ms = _graph_ms(dh_step, flush, max(args.steps, 10))
        dense_dh_ms = _graph_ms(lambda: torch.matmul(dY, W2.t()), flush, max(args.steps, 10))
        refh = (dY[:256].double() @ W2.double().t()) * (H[:256] > 0)
        errh = float((dH[:256].double() - refh).norm() / refh.norm().clamp_min(1e-30))
        del dH
        out["by_zero_ratio"][str(zr)] = {
            "value": round(eff / (ms * 1e-3) / 1e12, 2), "ms_per_step": round(ms, 4), "live_fraction": round(
                live / (tokens * d_ff), 4),
            "fwd_pit_m_TFLOPs": round(eff / 2 / (split[0] * 1e-3) / 1e12, 1),
            "bwd_pit_k_TFLOPs": round(eff / 2 / (split[1] * 1e-3) / 1e12, 1),
            "fwd_ms": round(split[0], 4), "bwd_ms": round(split[1], 4),
            "dH_sddmm": {"ms": round(dh_ms, 4), "effective_TFLOPs": round(eff / 2 / (dh_ms * 1e-3) / 1e12, 1),
                         "dense_cublas_ms": round(dense_dh_ms, 4), "rel_err_rows0_255_vs_f64": errh,
                         "execution": "CUDA graph: run_sddmm_like(dY, W2^T, H, (1,32), gate=H): both output indexes detected from H on the device + the SDDMM"},
            "fwd_path": "high-sparsity supergroup products + ordered partial-row reduction"
                        if live * 48 <= tokens * d_ff else "masked dense tiles on CTA pairs",
            "max_rel_err_vs_f64": err,
            "graph_replay_equals_eager": bool(torch.equal(O_g[0], Y) and torch.equal(O_g[1], dW2))}
        del H, keep
    first = out["by_zero_ratio"][str(zeros[0])]
    out["value"], out["ms_per_step"] = first["value"], first["ms_per_step"]
    return out


def c1_fp32_bench(args, dev, peaks):
    """BASELINE configs[0] on the GPU: 1024^3 fp32 (TF32 never used: K7 FFMA path, 1e-5 parity),
    detection from values + SpMM as one CUDA graph, L2 flushed. The reference's own number for this
    configuration is its CPU time (cpu_baseline, attached by run_ours)."""
    import torch

    from paper_2301_10936_b200.graph import CapturedSparseMatmul

    w = dict(C1_1024, name="c1_fp32_1024")
    g = torch.Generator(device=dev).manual_seed(3)
    keep = torch.rand((w["K"], w["M"] // 32), device=dev, generator=g) >= w["zero"]
    At = torch.randn((w["K"], w["M"]), device=dev, dtype=torch.float32, generator=g)
    At.mul_(keep.repeat_interleave(32, dim=1).float())
    A = At.t()
    B = torch.randn((w["K"], w["N"]), device=dev, dtype=torch.float32, generator=g)
    eff = 2.0 * w["N"] * int(keep.sum().item()) * 32
    plan = make_plan(w)
    eager = pit_run(plan, A, B, w)
    ref = A.double() @ B.double()
    err = float((eager.double() - ref).norm() / ref.norm())
    captured = CapturedSparseMatmul(plan, A, B)
    for _ in range(max(3, args.warmup)):
        captured.replay()
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    ev = []
    for _ in range(max(10, args.steps)):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        captured.replay()
        e1.record(stream)
        ev.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    return {"workload": w["desc"], "value": round(eff / (ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s (effective)",
            "ms_per_step": round(ms, 4), "dtype": "f32", "kernel": "spmm_simt (K7 FFMA, fp32, no TF32)",
            "rel_err_normwise_vs_f64": err, "tolerance": 1e-5,
            "graph_replay_equals_eager": bool(torch.equal(captured.C, eager)),
            "gpu_launches_per_step": captured.kernels_per_replay,
            "execution": "CUDA graph: build_index_from_tensor (32,1) + run_matmul_with_index (pit:k)"}


def e2e_ours(args, w, A, B, plan, eff_flops):
    """Host pinned A, B -> H2D -> detection -> SpMM -> D2H of C, all inside the timed region."""
    import torch

    import paper_2301_10936_b200 as pit

    Ah = torch.empty(A.t().shape, dtype=A.dtype, pin_memory=True) if w["axis"] == "k" else \
        torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
    Ah.copy_(A.t() if w["axis"] == "k" else A)
    Bh = torch.empty(B.shape, dtype=B.dtype, pin_memory=True)
    Bh.copy_(B)
    stream = torch.cuda.current_stream()

    def once():
        # public API on host buffers: A is uploaded for online detection; run_matmul_with_index then
        # streams B column slabs up, runs the SpMM per slab and streams C slabs down (3 streams)
        Ad = Ah.to("cuda", non_blocking=True)
        Ad = Ad.t() if w["axis"] == "k" else Ad
        idx = pit.build_index_from_tensor(Ad, w["micro"], w["axis"])
        C = pit.run_matmul_with_index(plan, pit.DenseTensor(Ad), pit.DenseTensor(Bh), idx)
        assert not C.array.is_cuda

    for _ in range(max(1, args.warmup)):
        once()
    torch.cuda.synchronize()
    n = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        once()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    return {"value": round(eff_flops / (ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": Ah.numel() * 2 + Bh.numel() * 2, "d2h_bytes_per_step": w["M"] * w["N"] * 2,
            "api": "build_index_from_tensor + run_matmul_with_index on pinned host buffers (B/C slabs pipelined)"}


# --------------------------------------------------------------------------- CPU baselines
# The reference's own CPU path, timed on the host cores beside the GPU numbers: `pittile` itself
# from baseline/_ref (the unmodified reference, installed offline: kind "reference") or, when that
# is absent, its restatement oracle/pit_oracle.py (kind "port"). Every sample runs in a fresh
# process (`bench.py --cpu-sections ...`) that never touches CUDA, so its fork pool is safe; the
# work is split over processes by independent units (M-block groups, sequences, heads' query
# blocks, experts) with no reduction, and each process runs the reference single-threaded
# (OPENBLAS_NUM_THREADS=1, workers=1: its fastest configuration).
REF_SITE = ROOT / "baseline" / "_ref"
MM_EXPR = "C[m,n] += A[m,k] * B[k,n]"
REF_TILES = {(16, 32, 128), (8, 32, 128), (32, 64, 32), (32, 32, 32)}  # reference tiles.py:106-116
_CPU = {}


def ref_backend():
    """pittile from baseline/_ref, or None."""
    if "backend" not in _CPU:
        P = None
        if (REF_SITE / "pittile").is_dir():
            sys.path.insert(0, str(REF_SITE))
            try:
                import pittile as P
            except Exception:
                P = None
        _CPU["backend"] = P
    return _CPU["backend"]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def ref_tile(axis: str, tile) -> tuple:
    """The reference registry has no B200 tile shapes; those run on the reference tile of the same
    PIT role (its default (32,64,32) for k and dense, (16,32,128) for m)."""
    tile = tuple(tile)
    if tile in REF_TILES:
        return tile
    return (16, 32, 128) if axis == "m" else (32, 64, 32)


def cpu_mm(A, B, axis, tile):
    """One product through the reference's public path: detection on the values
    (build_index_from_tensor, index.py:164-173) + run_matmul_with_index (executor.py:464-516).
    A must already be in the plan's layout (column-major for pit:k)."""
    P = ref_backend()
    if P is None:
        from oracle import pit_oracle as orc

        if axis == "dense":
            return orc.matmul_dense(A, B, tile)
        micro = (tile[0], 1) if axis == "k" else (1, tile[1])
        _, groups = orc.build_index_from_values(A, micro, axis)
        return (orc.matmul_pit_k if axis == "k" else orc.matmul_pit_m)(A, B, groups, micro, tile)
    key = (A.shape, B.shape[1], axis, tile)
    plan = _CPU.setdefault("plans", {}).get(key)
    if plan is None:
        expr = P.bind_extents(P.parse_expr(MM_EXPR), dict(m=A.shape[0], k=A.shape[1], n=B.shape[1]))
        plan = _CPU["plans"][key] = P.forced_plan(expr, axis, P.register_builtin_kernels(), tile_shape=tile)
    idx = None if axis == "dense" else P.build_index_from_tensor(A, plan.micro_tile, axis)
    return P.run_matmul_with_index(plan, P.DenseTensor(A), P.DenseTensor(B), idx).array


def _relu_mask(rng, shape, gran, zero):
    keep = rng.random((shape[0] // gran[0], shape[1] // gran[1])) >= zero
    return np.kron(keep, np.ones(gran, dtype=bool))


def cpu_job(name: str, rng):
    """(units_total, make_unit(i) -> unit data, run(unit) -> work, unit name, work unit, sample text)
    for one section. Units are generated before the timed region."""
    if name in WORKLOADS or name == "c1_1024":
        w = dict(WORKLOADS.get(name, C1_1024), name=name)
        M, K, N, t0 = w["M"], w["K"], w["N"], w["micro"][0]
        tile = ref_tile(w["axis"], w["tile"])
        B = rng.standard_normal((K, N), dtype=np.float32)
        if w["axis"] == "k":
            def make(i):
                A = rng.standard_normal((t0, K), dtype=np.float32) * _relu_mask(rng, (t0, K), (t0, 1), w["zero"])
                return np.asfortranarray(A)

            total, what = M // t0, f"{t0}-row M-block groups (all K, all N)"
        elif name.startswith("bert"):
            def make(i):
                A = rng.standard_normal((128, K), dtype=np.float32)
                A[int(rng.integers(16, 129)):] = 0.0
                return A

            total, what = M // 128, "sequences (128 padded rows each)"
        else:
            def make(i):
                return rng.standard_normal((128, K), dtype=np.float32) * _relu_mask(rng, (128, K), w["micro"], w["zero"])

            total, what = M // 128, "128-row slabs (all K, all N)"

        def run(A):
            cpu_mm(A, B, w["axis"], tile)
            return 2.0 * N * np.count_nonzero(A)

        return total, make, run, "TFLOP/s", 1e12, f"{what} of {name}, fp32, plan tile {tile}"
    if name == "attention":
        heads, seq, hd = 12, 4096, 64
        blocks = longformer_blocks(heads, seq, np.random.default_rng(5))  # [heads, seq/32, seq/64]
        V = rng.standard_normal((seq, hd), dtype=np.float32)

        def make(i):
            h, qb = divmod(i, seq // 32)
            live = np.repeat(blocks[h, qb], 64)
            return np.asfortranarray(rng.random((32, seq), dtype=np.float32) * live)

        def run(P):
            cpu_mm(P, V, "k", (32, 64, 32))
            return 2.0 * hd * np.count_nonzero(P)

        return heads * seq // 32, make, run, "TFLOP/s", 1e12, \
            "32-row query blocks of P.V (12 heads x 4096^2, 32x64 block mask), pit:k (32,1), fp32"
    if name == "opt_ffn2":
        tokens, d_ff, d_model, zero = 4096, 8192, 2048, 0.9
        W2 = rng.standard_normal((d_ff, d_model), dtype=np.float32)
        dY = rng.standard_normal((tokens, d_model), dtype=np.float32)

        def make(i):
            if i % 9 == 0:   # forward: 128 token rows of H, pit:m (1,32) -- 1/32 of the forward product
                return ("m", rng.random((128, d_ff), dtype=np.float32) * _relu_mask(rng, (128, d_ff), (1, 32), zero))
            # weight gradient: 32 neurons of H^T (all tokens), pit:k (32,1) on H^T column-major -- 1/256 of it
            return ("k", np.asfortranarray(rng.random((32, tokens), dtype=np.float32) *
                                           _relu_mask(rng, (tokens, 32), (1, 32), zero).T))

        def run(u):
            axis, A = u
            if axis == "m":
                cpu_mm(A, W2, "m", (16, 32, 128))
            else:
                cpu_mm(A, dY, "k", (32, 64, 32))
            return 2.0 * d_model * np.count_nonzero(A)

        return tokens // 128 + d_ff // 32, make, run, "TFLOP/s", 1e12, \
            "units of the step (1 forward 128-token slab, pit:m (1,32) H.W2, per 8 weight-grad 32-neuron slabs, " \
            "pit:k (32,1) H^T.dY: equal FLOPs), 90% zero, fp32"
    if name == "moe":
        d_model, d_ff, per_expert = 768, 3072, 128

        def make(i):
            return (rng.standard_normal((per_expert, d_model), dtype=np.float32),
                    rng.standard_normal((d_model, d_ff), dtype=np.float32) * 0.03,
                    rng.standard_normal((d_ff, d_model), dtype=np.float32) * 0.03)

        def run(u):
            x, w1, w2 = u
            h = np.maximum(cpu_mm(x, w1, "dense", (32, 64, 32)), 0.0)
            cpu_mm(np.ascontiguousarray(h, dtype=np.float32), w2, "dense", (32, 64, 32))
            return float(per_expert)

        return 128, make, run, "tokens/s", 1.0, \
            "experts of the 128-expert layer (128 tokens each = 16384 tokens), FFN1+ReLU+FFN2 on the dense plan, fp32"
    raise ValueError(name)


def _cpu_run_units(ids):
    run, units = _CPU["run"], _CPU["units"]
    return sum(run(units[i]) for i in ids)


def cpu_sample(name: str, procs: int, target_s: float, seed: int = 7) -> dict:
    """Time the reference path on a bounded sample of one section's units with `procs` processes."""
    import multiprocessing as mp

    rng = np.random.default_rng(seed)
    total, make, run, unit, scale, what = cpu_job(name, rng)
    _CPU["run"] = run
    _CPU["units"] = [make(0)]
    t = time.perf_counter()
    _cpu_run_units([0])
    per_unit = time.perf_counter() - t
    n = int(min(total, max(procs, target_s * procs / max(per_unit, 1e-4))))
    n = -(-n // procs) * procs if n >= procs else n
    n = min(n, total)
    _CPU["units"] = [make(i) for i in range(n)]
    # small workloads: the whole unit set repeated until the sample is long enough to time
    reps = max(1, int(target_s * procs / max(per_unit * n, 1e-6))) if n == total else 1
    chunks = [[j % n for j in range(i, n * reps, procs)] for i in range(procs)]
    if procs == 1:
        t = time.perf_counter()
        work = _cpu_run_units(chunks[0])
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            pool.map(_cpu_run_units, [[0]] * procs)  # warm the workers (imports, BLAS init)
            t = time.perf_counter()
            work = sum(pool.map(_cpu_run_units, chunks))
    secs = time.perf_counter() - t
    _CPU["units"] = []
    P = ref_backend()
    return {"value": round(work / secs / scale, 6 if scale > 1 else 1), "unit": unit, "cores": procs,
            "kind": "reference" if P is not None else "port", "seconds": round(secs, 2),
            "sample": f"{n} of {total} {what}" + (f", x{reps} passes" if reps > 1 else ""),
            "implementation": (f"pittile {P.__version__} (the reference, baseline/_ref) public API"
                               if P is not None else "oracle/pit_oracle.py restatement"),
            "cpu_model": cpu_model()}


def cpu_sections(names, target_s: float) -> dict:
    """Each section: the reference path on one core and on every host core."""
    out = {}
    cores = host_cores()
    for name in names:
        try:
            one = cpu_sample(name, 1, target_s)
            allc = cpu_sample(name, cores, target_s) if cores > 1 else one
            out[name] = dict(allc, single_core=one)
        except Exception as e:  # a CPU sample never costs the GPU line
            out[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
    return out


def cpu_sections_subprocess(names, target_s: float, timeout: float = 600) -> dict:
    """cpu_sections in a fresh interpreter (no CUDA context in the forking process)."""
    import subprocess

    r = subprocess.run([sys.executable, str(Path(__file__).resolve()), "--cpu-sections", ",".join(names),
                        "--cpu-seconds", str(target_s)], capture_output=True, text=True, timeout=timeout,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    try:
        return json.loads(r.stdout.strip().splitlines()[-1])
    except (ValueError, IndexError):
        return {n: {"error": (r.stderr or "no output")[-300:]} for n in names}


def base_config(w: dict, world: int = 1) -> dict:
    """The workload both arms run (identical dicts; each arm's dtype and execution are top-level)."""
    return {"workload": w["desc"].replace(" bf16", ""), "name": w["name"], "M": w["M"], "K": w["K"], "N": w["N"],
            "micro_tile": list(w["micro"]), "pit_axis": w["axis"], "zero_ratio": w["zero"],
            "plan_tile": list(w["tile"]), "parallelism": f"replica x{world} (per-GPU work fixed)",
            "l2": "inputs exceed L2; the GPU arm also flushes L2 (256 MiB write) before every step"}


def run_reference(args, w):
    """--impl reference: the reference's own CPU path on every host core, same workload/config."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    cores = host_cores()
    vals, base = [], None
    for i in range(args.warmup + args.steps):
        r = cpu_sample(w["name"], cores, args.ref_seconds, seed=7 + i)
        if i >= args.warmup:
            vals.append(r["value"])
            base = r
    value = statistics.mean(vals)
    # one step = the full workload (every M-block group); its expected effective FLOPs / the rate
    step_flops = 2.0 * w["M"] * w["K"] * w["N"] * (1.0 - (w["zero"] or 0.0))
    cfg = base_config(w, world)
    return {
        "impl": "reference", "metric": "PIT sparse matmul effective TFLOP/s (online detection + SpMM)",
        "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(step_flops / (value * 1e12) * 1e3, 1) if value > 0 else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": cfg,
        "execution": f"reference CPU path ({base['implementation']}), {cores} processes x 1 thread, fp32 "
                     "(the reference has no bf16, executor.py:40-41)",
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample", "implementation",
                                               "cpu_model")} | {"value": round(value, 6)},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-index-bench", action="store_true")
    ap.add_argument("--no-moe", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the micro-tile x sparsity sweep")
    ap.add_argument("--no-attn", action="store_true", help="skip the C3 block-sparse attention section")
    ap.add_argument("--no-bert", action="store_true", help="skip the C2 BERT varlen FFN1 section")
    ap.add_argument("--no-opt", action="store_true", help="skip the C4 OPT FFN2 section")
    ap.add_argument("--no-graph", action="store_true", help="time eager API calls instead of the captured step")
    ap.add_argument("--no-c1", action="store_true", help="skip the BASELINE configs[0] (1024^3 fp32) section")
    ap.add_argument("--cpu-seconds", type=float, default=3.0, help="target seconds per CPU-baseline sample")
    ap.add_argument("--cpu-sections", default=None, help=argparse.SUPPRESS)  # internal: CPU samples, no CUDA
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    args = ap.parse_args()
    if args.cpu_sections:
        print(json.dumps(cpu_sections(args.cpu_sections.split(","), args.cpu_seconds)), flush=True)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (the driver may also launch it so)
        import socket

        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    w = dict(WORKLOADS[args.workload], name=args.workload)
    res = run_reference(args, w) if args.impl == "reference" else run_ours(args, w)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
