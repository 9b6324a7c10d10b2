"""Multi-process plumbing of the N>1 path on CPU (gloo, world_size 2): the
NCCL-id hand-off used by the expert-parallel engine and the max-over-ranks
timing reduction in bench.py, plus the expert-shard bookkeeping the engine
applies per layer (destination-major labels, send/receive segments)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ident = bench.share_ep_id(rank, world, lambda: "ab" * 128)
    slowest = bench.max_over_ranks(10.0 + rank, world, torch.device("cpu"))
    q.put((rank, ident, slowest))
    dist.destroy_process_group()


def test_ep_id_handoff_and_max_over_ranks_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert {o[1] for o in out} == {"ab" * 128}
    assert all(o[2] == 11.0 for o in out)


def _shard_exchange(idx_per_rank, E, G):
    """Python restatement of the engine's per-layer EP bookkeeping
    (engine_ep.cpp): destination-major labels, stable sort, per-destination
    counts, receive layout, local stable sort, return and un-permute."""
    El = E // G
    label = np.array([(e % G) * El + e // G for e in range(E)])
    sends = []
    for r, idx in enumerate(idx_per_rank):
        lbl = label[idx.ravel()]
        order = np.argsort(lbl, kind="stable")
        counts = np.bincount(lbl, minlength=E)
        sends.append((order, counts))
    recv = {}
    for dst in range(G):
        rows, ids = [], []
        for src in range(G):
            order, counts = sends[src]
            off = counts[: dst * El].sum()
            seg = order[off: off + counts[dst * El:(dst + 1) * El].sum()]
            rows += [(src, int(x)) for x in seg]
            for j in range(El):
                ids += [j] * int(counts[dst * El + j])
        recv[dst] = (rows, np.array(ids))
    return label, sends, recv


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_expert_shard_exchange_covers_every_routed_row_once(G):
    E, k, T = 8, 2, 37
    rng = np.random.default_rng(G)
    idx = [np.stack([rng.permutation(E)[:k] for _ in range(T)]) for _ in range(G)]
    label, sends, recv = _shard_exchange(idx, E, G)
    seen = set()
    for dst, (rows, ids) in recv.items():
        for (src, flat), j in zip(rows, ids):
            e = int(idx[src].ravel()[flat])
            assert e % G == dst and e // G == j  # the owner rank, as its local expert
            seen.add((src, flat))
    assert len(seen) == G * T * k
