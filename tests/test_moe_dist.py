"""CPU, world size 2 over gloo: the expert-parallel exchanges of SwitchMoE equal the single-process
oracle. "default" on a group whose ranks cannot map each other's regions: every rank falls back to
the all-to-all-v exchange together. "nccl": counts all-to-all, token all-to-all-v, receive plan,
reverse all-to-all, gate-scaled combine. "peer": the peer-memory protocol of csrc/pit_ep.cu (region positions, receive plan, pull
combine) restated on CPU (tests/moe_oracle_backend.EmulatedPeerExchange). Compute runs in the
test-only oracle backend."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pit_oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(T, E, d, F, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((2 * T, d)).astype(np.float32)
    logits = rng.standard_normal((2 * T, E)).astype(np.float32)
    w1 = (rng.standard_normal((E, d, F)) / np.sqrt(d)).astype(np.float32)
    w2 = (rng.standard_normal((E, F, d)) / np.sqrt(F)).astype(np.float32)
    return x, logits, w1, w2


def _unmappable_peers(group, *args):
    """A PeerExchange whose IPC open fails on rank 1 only: like PeerExchange, the ranks share their
    errors and all raise PeerUnavailable together."""
    from paper_2301_10936_b200.moe import PeerUnavailable

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    errs = [None] * world
    dist.all_gather_object(errs, "cudaIpcOpenMemHandle: peer access unsupported" if rank == 1 else "", group=group)
    bad = [(r, e) for r, e in enumerate(errs) if e]
    raise PeerUnavailable(f"peer-memory exchange unavailable (rank {bad[0][0]}: {bad[0][1]})")


def _worker(rank, world, port, T, E, d, F, q, exchange="nccl"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from moe_oracle_backend import EmulatedPeerExchange, OracleBackend
        from paper_2301_10936_b200.moe import SwitchMoE

        x, logits, w1, w2 = _problem(T, E, d, F, seed=5)
        El = E // world
        sl = slice(rank * T, (rank + 1) * T)
        factory = EmulatedPeerExchange if exchange == "peer" else _unmappable_peers if exchange == "default" else None
        layer = SwitchMoE(torch.from_numpy(w1[rank * El : (rank + 1) * El]).double(),
                          torch.from_numpy(w2[rank * El : (rank + 1) * El]).double(), E, group=dist.group.WORLD,
                          backend=OracleBackend(), exchange=None if exchange == "default" else exchange,
                          exchange_factory=factory)
        out = layer(torch.from_numpy(x[sl]).double(), torch.from_numpy(logits[sl]))
        received = layer.stats.received
        if exchange == "default":  # no peer mappings: every rank fell back to the all-to-all-v exchange
            assert layer.exchange == "nccl" and "rank 1" in layer.fallback_reason
            out2 = layer(torch.from_numpy(x[sl]).double(), torch.from_numpy(logits[sl]))
            assert torch.equal(out, out2)
        if exchange == "peer":
            received = int(layer._peer.lcounts.sum())
            out2 = layer(torch.from_numpy(x[sl]).double(), torch.from_numpy(logits[sl]))  # regions reused
            assert torch.equal(out, out2)
        q.put((rank, out.numpy(), received))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["nccl", "peer", "default"])
@pytest.mark.parametrize("E", [4, 8])
def test_expert_parallel_exchange_matches_single_process(E, exchange):
    T, d, F, world = 37, 16, 24, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, E, d, F, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict((r, (o, n)) for r, o, n in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, logits, w1, w2 = _problem(T, E, d, F, seed=5)
    ref = orc.switch_forward(x, logits, w1, w2)
    got = np.concatenate([results[0][0], results[1][0]])
    assert orc.max_rel_error(got, ref) <= 1e-6  # gate is carried in float32
    assert results[0][1] + results[1][1] == 2 * T  # every token computed exactly once (dropless)
