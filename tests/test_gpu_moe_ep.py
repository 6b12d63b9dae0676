"""Expert-parallel MoE over peer memory (csrc/pit_ep.cu) on the GPU.

* one rank: the dispatch / receive-plan / signal / combine kernels run against the rank's own
  region; the layer equals the f64 oracle within the bf16 gate and the NCCL-path result bitwise
  (both round the expert output to bf16 before the gate, SWrite * gate in fp32);
* the whole layer captured in one CUDA graph replays bitwise equal to the eager call (no host
  synchronisation anywhere on the path);
* two ranks on the one visible GPU (two processes, gloo for the IPC handle exchange): the real
  cross-process protocol — IPC-mapped regions, epoch flags, pulls — against the single-process oracle,
  over several consecutive layers (buffer reuse), with no timed-out wait."""

import os
import socket

import numpy as np
import pytest

from oracle import pit_oracle as orc

pytestmark = pytest.mark.gpu


def _bf16_round(a):
    import torch

    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def _problem(T, E, d, F, seed, skew=0.0):
    rng = np.random.default_rng(seed)
    x = _bf16_round(rng.standard_normal((T, d)))
    logits = rng.standard_normal((T, E)).astype(np.float32)
    logits[:, 0] += skew
    w1 = _bf16_round(rng.standard_normal((E, d, F)) / np.sqrt(d))
    w2 = _bf16_round(rng.standard_normal((E, F, d)) / np.sqrt(F))
    return x, logits, w1, w2


def _cuda(a, dtype=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.to(dtype) if dtype is not None else t


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("T,E,d,F,skew", [(1000, 8, 256, 512, 0.0), (4096, 128, 768, 3072, 0.0),
                                          (3000, 16, 128, 256, 3.0), (5, 4, 64, 128, 0.0)])
def test_peer_exchange_one_rank(T, E, d, F, skew):
    import torch
    import torch.distributed as dist

    from paper_2301_10936_b200.moe import SwitchMoE

    x, logits, w1, w2 = _problem(T, E, d, F, seed=T + E, skew=skew)
    xd, ld = _cuda(x, torch.bfloat16), _cuda(logits)
    layer = SwitchMoE(_cuda(w1, torch.bfloat16), _cuda(w2, torch.bfloat16), E, exchange="peer")
    try:
        out = layer(xd, ld)
        out2 = layer(xd, ld)  # second epoch through the same region
        torch.cuda.synchronize()
        assert layer._peer.error() == 0
        assert torch.equal(out, out2)
        ref = orc.switch_forward(x, logits, w1, w2, round_hidden=_bf16_round)
        assert orc.max_rel_error(out.float().cpu().numpy(), ref) <= 1e-2
        # the NCCL-path orchestration (single-rank group) computes the same bf16 values
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1)
        try:
            nccl = SwitchMoE(layer.w1, layer.w2, E, group=dist.group.WORLD, exchange="nccl")
            assert torch.equal(nccl(xd, ld), out)
        finally:
            dist.destroy_process_group()
    finally:
        layer.close()


def test_peer_layer_in_one_cuda_graph():
    import torch

    from paper_2301_10936_b200.moe import SwitchMoE

    x, logits, w1, w2 = _problem(2048, 16, 256, 512, seed=9)
    xd, ld = _cuda(x, torch.bfloat16), _cuda(logits)
    layer = SwitchMoE(_cuda(w1, torch.bfloat16), _cuda(w2, torch.bfloat16), 16, exchange="peer")
    try:
        eager = layer(xd, ld).clone()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            layer(xd, ld)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = layer(xd, ld)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager)
        # new inputs through the captured graph: same as eager on them
        xd.copy_(torch.flip(xd, dims=[0]))
        g.replay()
        torch.cuda.synchronize()
        got = out.clone()
        assert torch.equal(got, layer(xd, ld))
        assert layer._peer.error() == 0
    finally:
        layer.close()


def _ep_worker(rank, world, port, T, E, d, F, layers, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2301_10936_b200.moe import SwitchMoE

        x, logits, w1, w2 = _problem(world * T, E, d, F, seed=21, skew=1.0)
        El = E // world
        sl = slice(rank * T, (rank + 1) * T)
        layer = SwitchMoE(_cuda(w1[rank * El:(rank + 1) * El], torch.bfloat16),
                          _cuda(w2[rank * El:(rank + 1) * El], torch.bfloat16), E, group=dist.group.WORLD,
                          exchange="peer")
        outs = []
        for i in range(layers):
            # layer i sees a row-rotated batch: every epoch moves different rows through the regions
            xs = np.roll(x[sl], i, axis=0)
            ls = np.roll(logits[sl], i, axis=0)
            outs.append(layer(_cuda(xs, torch.bfloat16), _cuda(ls)).float().cpu().numpy())
        torch.cuda.synchronize()
        err = layer._peer.error()
        layer.close()
        q.put((rank, outs, err, None))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, -1, f"{type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_peer_exchange_two_processes_one_gpu():
    import torch.multiprocessing as mp

    T, E, d, F, world, layers = 600, 8, 128, 256, 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_worker, args=(r, world, port, T, E, d, F, layers, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        results = {}
        for _ in range(world):
            r, outs, err, msg = q.get(timeout=240)
            assert msg is None, msg
            assert err == 0, f"rank {r}: a peer wait timed out"
            results[r] = outs
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.exitcode is None:
                p.kill()
    x, logits, w1, w2 = _problem(world * T, E, d, F, seed=21, skew=1.0)
    for i in range(layers):
        xs = np.concatenate([np.roll(x[r * T:(r + 1) * T], i, axis=0) for r in range(world)])
        ls = np.concatenate([np.roll(logits[r * T:(r + 1) * T], i, axis=0) for r in range(world)])
        ref = orc.switch_forward(xs, ls, w1, w2, round_hidden=_bf16_round)
        got = np.concatenate([results[r][i] for r in range(world)])
        assert orc.max_rel_error(got, ref) <= 1e-2
