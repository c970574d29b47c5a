"""Row-sharded explicit step on ONE GPU: R virtual ranks stepped in lockstep
(LocalTransport: each phase for every rank, then copies between their buffers -- no rank waits
on another) against the single-GPU DeviceStepper.  Same kernels, same per-row order and a
replicated pressure solve with an identical right-hand side: the fields must be bitwise equal."""

import numpy as np
import pytest

import paper_2303_01760_b200 as hn
from paper_2303_01760_b200 import nodesets
from paper_2303_01760_b200 import sharded as S

pytestmark = pytest.mark.gpu


def _case(ns, Ra=1e6, seed=0, rbf_n=None):
    settings = hn.PoissonSolveSettings()
    ops = hn.build_operators(ns, {"wall:x-"}, settings, interior_rbf_n=rbf_n)
    params = hn.PhysicsParams(Ra, 0.71)
    dt = hn.TimeControls.from_spacing(float(np.min(ns.spacing)), 1.0, Ra=Ra).dt
    d = ns.dim
    T0 = (ns.positions[:, 0] - 0.5) + 1e-3 * np.random.default_rng(seed).normal(size=len(ns))
    st = hn.FieldState(np.zeros((len(ns), d)), np.zeros(len(ns)), T0)
    hn.apply_temperature_bc(st.temperature, ops)
    return ops, params, settings, dt, st


def _run_both(ns, world, steps, **kw):
    ops, params, settings, dt, st = _case(ns, **kw)
    single = hn.DeviceStepper(ops, params, settings, dt, st)
    tr = S.LocalTransport(world)
    ranks = [S.ShardedStepper(ops, params, settings, dt, st, r, world, transport=tr) for r in range(world)]
    for _ in range(steps):
        single.step()
        S.step_lockstep(ranks, tr)
    return single, ranks, tr


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_step_bitwise_equals_single_gpu_2d(world):
    ns = nodesets.hybrid_hole_2d(60, seed=2)
    single, ranks, tr = _run_both(ns, world, steps=12)
    want = single.state()
    for got in S.gather_states(ranks, tr):
        assert got.velocity.tobytes() == want.velocity.tobytes()
        assert got.temperature.tobytes() == want.temperature.tobytes()
        assert got.pressure.tobytes() == want.pressure.tobytes()
    lat = [r.latch_host() for r in ranks]
    assert all(int(l[0]) == 12 and l[1] == 0 and l[3] == 0 for l in lat)
    ranks[0].check_finite(lat)
    # each rank holds a slab plus a thin halo, not the whole set
    for r in ranks:
        assert r.plan.n_own <= -(-len(ns) // world)
        assert 0 < r.plan.n_halo < len(ns) // 3


def test_sharded_step_bitwise_equals_single_gpu_3d():
    ns = nodesets.hybrid_sphere_3d(18, seed=4, refine=2.8)  # the config-4 twin recipe, smaller
    single, ranks, tr = _run_both(ns, 2, steps=4, Ra=1e5, rbf_n=30)
    want = single.state()
    for got in S.gather_states(ranks, tr):
        assert got.velocity.tobytes() == want.velocity.tobytes()
        assert got.temperature.tobytes() == want.temperature.tobytes()


def test_sharded_divergence_latch_reports_global_node():
    """A non-finite temperature planted in one rank's rows shows up in the combined latch with
    its global node id, at the step the single-GPU stepper reports."""
    ns = nodesets.hybrid_hole_2d(40, seed=5)
    ops, params, settings, dt, st = _case(ns)
    bad = int(np.nonzero(ns.interior_mask)[0][-1])
    st.temperature[bad] = np.inf
    single = hn.DeviceStepper(ops, params, settings, dt, st)
    single.step()
    with pytest.raises(hn.SolverDivergenceError) as ref:
        single.check_finite()
    tr = S.LocalTransport(2)
    ranks = [S.ShardedStepper(ops, params, settings, dt, st, r, 2, transport=tr) for r in range(2)]
    S.step_lockstep(ranks, tr)
    with pytest.raises(hn.SolverDivergenceError) as got:
        ranks[0].check_finite([r.latch_host() for r in ranks])
    assert got.value.step == ref.value.step == 1
    assert got.value.node == ref.value.node


@pytest.mark.parametrize("case", ["2d", "3d"])
def test_row_sharded_weights_bitwise_equal_single_gpu(case):
    """compute_weights with the interior rows cut over 3 (virtual) ranks and all-gathered
    (SURVEY §8(e)): stencils and weights equal the single-GPU table bit for bit."""
    if case == "2d":
        ns, ops, rbf_n = nodesets.hybrid_hole_2d(60, seed=2), [hn.Laplacian(), hn.Partial(0), hn.Partial(1)], None
    else:
        ns = nodesets.hybrid_sphere_3d(18, seed=4)
        ops, rbf_n = [hn.Laplacian(), hn.Partial(0), hn.Partial(1), hn.Partial(2)], 20
    want = hn.compute_weights(ns, ops, rbf_n=rbf_n)
    world = 3
    tr = S.LocalTransport(world)
    shards = [S.WeightShard(ns, ops, r, world, rbf_n) for r in range(world)]
    assert sum(s.local["rbf"].K for s in shards) == shards[0].k_rbf
    for got in S.merge_weight_shards(shards, tr):
        assert np.array_equal(got.indices, want.indices)
        assert np.array_equal(got.sizes, want.sizes)
        assert np.array_equal(got.method, want.method)
        for op in ops:
            assert got.weights[op].tobytes() == want.weights[op].tobytes()
    # one real rank of a world of 1 goes through the same code
    one = S.compute_weights_sharded(ns, ops, 0, 1, S.LocalTransport(1), rbf_n)
    assert one.weights[ops[0]].tobytes() == want.weights[ops[0]].tobytes()
