"""Multi-rank path on CPU (gloo, world_size 2): the batch partitioner covers
every matrix exactly once, and sharded-then-all-reduced config-3 totals equal
the single-process totals.  Each rank computes its shard with the CPU oracle
as a stand-in for the CUDA sweeps (no GPU here); the partitioning and the
collective are the product code in paper_1902_10078_b200/dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1902_10078_b200.dist import reduce_totals, shard_bounds


@pytest.mark.parametrize("batch,world", [(256, 8), (7, 2), (3, 4), (1, 1), (0, 2)])
def test_shards_cover_batch_once(batch, world):
    seen = []
    for r in range(world):
        a, b = shard_bounds(batch, world, r)
        assert 0 <= a <= b <= batch
        seen.extend(range(a, b))
    assert seen == list(range(batch))
    sizes = [np.subtract(*shard_bounds(batch, world, r)[::-1]) for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, L, y, tau2, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as orc
    a, b = shard_bounds(L.shape[0], world, rank)
    loss, lbar, tbar, st, _ = orc.Oracle("restatement").marginal_likelihood_grad(L[a:b], y[a:b], tau2)
    tot = reduce_totals([torch.from_numpy(loss), torch.from_numpy(tbar)])
    out[rank] = tot.numpy().copy()
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_allreduce_matches_single_process(oracle):
    from tests import common as cm
    rng = np.random.default_rng(3)
    B, n, k, tau2 = 5, 300, 4, 0.01
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(0, 1, (B, n))
    loss, _, tbar, st, _ = oracle.marginal_likelihood_grad(L, y, tau2)
    want = np.array([loss.sum(), tbar.sum()])
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), L, y, tau2, out), nprocs=world, join=True)
    for r in range(world):
        np.testing.assert_allclose(out[r], want, rtol=1e-13)


def _bench_worker(rank, world, port, out):
    """bench.py's strong-scaling arithmetic: each rank's slice of the batch,
    the max-over-ranks step time, B_total * n / that time."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    a, b = bench.strong_slice(256, world, rank)
    local_ms = 1.0 + rank  # rank 1 is the slow one
    ms = bench.rank_max(local_ms, "cpu")
    out[rank] = (a, b, ms, 256 * 65536 / (ms / 1e3))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_strong_split_and_rank_max():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_bench_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert (out[0][0], out[0][1], out[1][0], out[1][1]) == (0, 128, 128, 256)
    assert out[0][2] == out[1][2] == 2.0  # both ranks report the slowest rank's time
    assert out[0][3] == 256 * 65536 / 2e-3
