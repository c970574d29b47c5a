"""N>1 host logic of bench.py on CPU with gloo, world_size 2 (one process per rank, as
torchrun launches it): weak-scaling shards are independent node sets of equal size,
and the reported time is the max over ranks.  The path has no data-path collective:
weight computation shards by node set."""

import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import numpy as np
    import bench
    r, w = bench.dist_init(world)
    assert (r, w) == (rank, world)
    ns = bench.build_nodeset(1, bench.shard_seed(0, r))
    local = float(10 + 5 * r)  # pretend per-rank step time
    t = bench.max_over_ranks(local, w)
    bench.barrier(w)
    out[rank] = (t, len(ns), float(np.sum(ns.positions[:100])))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_weak_scaling_shards_and_max_over_ranks():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 15.0          # max over ranks on every rank
    assert res[0][1] == res[1][1] == 99856         # equal per-rank work (weak scaling)
    assert res[0][2] != res[1][2]                  # independent node sets


def test_reference_arm_runs_only_on_rank0(monkeypatch):
    sys.path.insert(0, str(ROOT))
    import bench

    class A:
        config = 0
        steps = 1
        warmup = 0

    assert bench.run_reference(A(), rank=1, world=2) is None
