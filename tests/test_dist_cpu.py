"""Multi-rank plumbing of bench.py on CPU (gloo, world size 2): disjoint
right-hand-side sharding (weak scaling, no data-path collective) and the
max-over-ranks / sum-over-ranks reductions used for the timed value."""

import os
import socket

import pytest
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    d = bench.Dist("gloo")
    cols = [bench.shard_columns(s, d.rank, d.world, 16) for s in range(8)]
    t_max = d.max(10.0 + d.rank)     # a per-rank "elapsed time"
    it_sum = d.sum(100 + d.rank)     # per-rank iteration counts
    d.barrier()
    d.close()
    q.put((rank, cols, t_max, it_sum))


@pytest.mark.timeout(120)
def test_two_rank_sharding_and_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (c, t, s)) for r, c, t, s in (q.get(timeout=100) for _ in procs))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    c0, c1 = out[0][0], out[1][0]
    assert not set(c0) & set(c1)                    # disjoint columns per rank
    assert sorted(c0 + c1) == list(range(16))       # 8 steps x 2 ranks cover the 16 rhs once
    assert out[0][1] == out[1][1] == 11.0           # time = max over ranks
    assert out[0][2] == out[1][2] == 201.0          # work = sum over ranks


def _setup_worker(rank, world, port, q):
    import types

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    d = bench.Dist("gloo")
    P = bench.build_shared(types.SimpleNamespace(config="1", cstab="cache"), d)
    d.close()
    q.put((rank, float(P.rhs.sum()), int(P.forms.helmholtz.nnz), int(P.coarse.m_total)))


@pytest.mark.timeout(300)
def test_two_rank_shared_setup():
    """bench.build_shared: rank 0 builds the host setup once, rank 1 loads it."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_setup_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, rest) for r, *rest in (q.get(timeout=280) for _ in procs))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    assert out[0] == out[1]
