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


# ---------------------------------------------------------------- row-sharded step: halo plan
def _stencil_graph(n=600, k=7, seed=0):
    """Random 2D nodes with k-nearest stencils: (positions, rows, cols) of every reference."""
    import numpy as np
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 2))
    _, idx = cKDTree(pos).query(pos, k=k)
    rows = np.repeat(np.arange(n), k)
    return pos, rows, idx.ravel().astype(np.int64)


def _pack(plan, block, ncomp):
    return block.reshape(-1)[plan.pack_map(ncomp, block.shape[1])].copy()


def _unpack(plan, block, ncomp, recv):
    block.reshape(-1)[plan.unpack_map(ncomp, block.shape[1])] = recv


def test_halo_plans_agree_across_ranks_and_cover_every_column():
    import numpy as np
    sys.path.insert(0, str(ROOT))
    from paper_2303_01760_b200 import sharded as S
    pos, rows, cols = _stencil_graph()
    for world in (1, 2, 3, 5):
        owner = S.partition_nodes(pos, world)
        counts = np.bincount(owner, minlength=world)
        assert counts.max() - counts.min() <= 1                       # equal-count slabs
        plans = [S.build_halo_plan(owner, rows, cols, r, world) for r in range(world)]
        for r, pl in enumerate(plans):
            assert np.array_equal(np.sort(pl.own_glob), np.nonzero(owner == r)[0])
            assert not np.intersect1d(pl.own_glob, pl.halo_glob).size
            mine = owner[rows] == r
            assert (pl.glob2loc[cols[mine]] >= 0).all()               # every column a row reads is local
            assert np.array_equal(pl.loc2glob[pl.glob2loc[pl.loc2glob]], pl.loc2glob)
            for p in range(world):                                    # my send list == p's halo group from me
                assert pl.send_counts[p] == plans[p].recv_counts[r]
            assert pl.send_counts[r] == 0 and pl.recv_counts[r] == 0
        # a lockstep exchange of a 3-plane SoA field fills every halo with the owner's values
        f = np.random.default_rng(1).normal(size=(3, len(pos)))
        import torch
        blocks = [f[:, pl.loc2glob].copy() for pl in plans]
        for b, pl in zip(blocks, plans):
            b[:, pl.n_own:] = np.nan
        parts = [(pl, torch.from_numpy(_pack(pl, b, 3)), torch.empty(pl.n_halo * 3, dtype=torch.float64), 3)
                 for pl, b in zip(plans, blocks)]
        S.LocalTransport(world).halo(parts)
        for (pl, _, recv, _), b in zip(parts, blocks):
            _unpack(pl, b, 3, recv.numpy())
            assert np.array_equal(b, f[:, pl.loc2glob])
        # the padded all-gather of the owned rows rebuilds the global vector on every rank
        g = f[0]
        gparts = []
        for pl in plans:
            mine = torch.zeros(pl.max_own, dtype=torch.float64)
            mine[: pl.n_own] = torch.from_numpy(g[pl.own_glob])
            gparts.append((mine, torch.empty(pl.max_own * world, dtype=torch.float64)))
        S.LocalTransport(world).gather(gparts)
        for pl, (_, out) in zip(plans, gparts):
            assert np.array_equal(out.numpy()[pl.gather_pos], g)


def _halo_worker(rank, world, port, out):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2303_01760_b200 import sharded as S
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, rows, cols = _stencil_graph(seed=3)
    owner = S.partition_nodes(pos, world)
    plan = S.build_halo_plan(owner, rows, cols, rank, world)
    tr = S.TorchDistTransport()
    f = np.random.default_rng(7).normal(size=(2, len(pos)))      # the same global field on every rank
    block = f[:, plan.loc2glob].copy()
    block[:, plan.n_own:] = np.nan                                 # halo unknown until exchanged
    recv = torch.empty(plan.n_halo * 2, dtype=torch.float64)
    tr.halo([(plan, torch.from_numpy(_pack(plan, block, 2)), recv, 2)])
    _unpack(plan, block, 2, recv.numpy())
    halo_ok = bool(np.array_equal(block, f[:, plan.loc2glob]))
    # one ELL-style gather pass on local numbering == the global pass on my rows
    mine = owner[rows] == rank
    loc = np.zeros(len(pos))
    np.add.at(loc, rows[mine], block[0][plan.glob2loc[cols[mine]]])
    glob = np.zeros(len(pos))
    np.add.at(glob, rows, f[0][cols])
    pass_ok = bool(np.array_equal(loc[plan.own_glob], glob[plan.own_glob]))
    mine_pad = torch.zeros(plan.max_own, dtype=torch.float64)
    mine_pad[: plan.n_own] = torch.from_numpy(glob[plan.own_glob])
    gathered = torch.empty(plan.max_own * world, dtype=torch.float64)
    tr.gather([(mine_pad, gathered)])
    gather_ok = bool(np.array_equal(gathered.numpy()[plan.gather_pos], glob))
    out[rank] = (halo_ok, pass_ok, gather_ok, int(plan.n_halo))
    dist.destroy_process_group()


def test_halo_exchange_and_row_gather_over_gloo_world2():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_halo_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        halo_ok, pass_ok, gather_ok, n_halo = res[r]
        assert halo_ok and pass_ok and gather_ok
        assert 0 < n_halo < 300          # a thin strip of the 600 nodes, not everything
