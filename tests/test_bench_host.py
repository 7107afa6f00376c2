"""Host-side logic of bench.py: the replica aggregation over ranks (world_size 2, gloo,
CPU), the clock-record parser and the oracle bounded-sample extraction."""
import json
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t, u = bench.reduce_over_ranks(dist, 10.0 + rank, 100.0 * (rank + 1))
    out[rank] = (t, u)
    dist.destroy_process_group()


def test_replica_reduction_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] == (11.0, 300.0)   # max time, summed work


def test_reduce_single_process():
    import bench
    assert bench.reduce_over_ranks(None, 5.0, 7.0) == (5.0, 7.0)


def test_oracle_sample_extraction_is_same_workload():
    import bench
    from workload import make_system
    prob, J, rhs = make_system(2, dims=(6, 5, 8))
    prob._config = 2
    res = bench.oracle_sample(J, prob, 10, restart=30, tol=1e-8)
    assert res["cores"] == 1 and res["value"] > 0 and "2 of 8 z-planes" in res["sample"]
