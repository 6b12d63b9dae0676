"""CPU: `bench.py --gpus N` without a torchrun environment re-launches itself as N ranks (one process
per GPU), and the reference arm under N ranks prints exactly one line, from rank 0, with n_gpus = N."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_bench_gpus_flag_spawns_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-seconds", "0.2"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_cpu_sections_one_and_all_cores():
    """The CPU baselines beside each bench section: the reference path (pittile from baseline/_ref when
    installed, else the oracle port) on one core and on every host core, CPU model stated."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--cpu-sections", "c1_1024,bert_ffn1",
                        "--cpu-seconds", "0.05"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for name in ("c1_1024", "bert_ffn1"):
        s = d[name]
        assert "error" not in s, s
        assert s["value"] > 0 and s["unit"] == "TFLOP/s" and s["kind"] in ("reference", "port")
        assert s["cores"] == len(os.sched_getaffinity(0)) and s["single_core"]["cores"] == 1
        assert s["cpu_model"]


def test_reference_arm_config_matches_ours():
    sys.path.insert(0, str(ROOT))
    import bench

    w = dict(bench.WORKLOADS[bench.DEFAULT_WORKLOAD], name=bench.DEFAULT_WORKLOAD)
    cfg = bench.base_config(w)
    for key in ("M", "K", "N", "micro_tile", "pit_axis", "zero_ratio", "plan_tile", "workload"):
        assert key in cfg
    assert "bf16" in cfg["workload"] or "fp32" not in cfg["workload"]
