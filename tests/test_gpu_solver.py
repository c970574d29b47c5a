"""GPU time stepping (solver.py), modelled on the reference's pkg/tests/test_solver.py,
plus parity with the reference's recorded steps (goldens) and with the oracle.

Tolerances: explicit kernels fed identical inputs are bit-exact vs the oracle; pressure
(direct-solve accurate) <= 1e-10 relative; fields after k steps <= 1e-8 relative
(north star).  The reference's run() drives node generation we do not ship, so run()
tests pass a node set."""

from types import SimpleNamespace

import numpy as np
import numpy.testing as npt
import pytest

import paper_2303_01760_b200 as hn
from oracle import hn_oracle as O
from paper_2303_01760_b200 import nodesets
from paper_2303_01760_b200.operators import FieldState
from paper_2303_01760_b200.solver import (DeviceStepper, PhysicsParams, PoissonSolveSettings, TimeControls,
                                          apply_temperature_bc, apply_velocity_bc, build_operators,
                                          interior_divergence, momentum_predict, nusselt_average, pressure_solve,
                                          run, temperature_step, velocity_correct)

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-8


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def tie_override(ns):
    """The reference's boundary stencils on the exact-tie rows."""
    bidx = np.nonzero(ns.boundary_mask)[0]
    t = hn.boundary_partial_table(ns, bidx, exclude=ns.boundary_mask)
    rows = np.asarray(t.tie_rows, dtype=np.int64)
    st = O.boundary_stencils(ns, rows, ns.boundary_mask, t.indices.shape[1]) if len(rows) else np.empty((0, 12))
    return rows, st


@pytest.fixture(scope="module")
def dvd_setup(golden):
    ns, g = golden("dvd_coarse")
    settings = PoissonSolveSettings()
    ops = build_operators(ns, {"wall:x-"}, settings, boundary_override=tie_override(ns))
    return ns, ops, PhysicsParams(1e6, 0.71), settings, g


class TestTimeControls:
    def test_dt_formula(self):
        assert TimeControls.from_spacing(0.01, 1.0).dt == pytest.approx(0.1 * 0.01 ** 2 / 2)

    def test_advective_cap_only_binds_when_coarse(self):
        assert TimeControls.from_spacing(0.005, 1.0, Ra=1e6).dt == pytest.approx(0.1 * 0.005 ** 2 / 2)
        assert TimeControls.from_spacing(0.04, 1.0, Ra=1e6).dt == pytest.approx(40.0 / 1e6)


class TestMomentumPredict:
    def test_quiescent_stays_quiescent(self, dvd_setup):
        ns, ops, params, _, _ = dvd_setup
        npt.assert_array_equal(momentum_predict(FieldState.zeros(len(ns), 2), ops, params, 1e-5), 0.0)

    def test_pure_buoyancy_kick(self, dvd_setup):
        ns, ops, params, _, _ = dvd_setup
        state = FieldState.zeros(len(ns), 2)
        state.temperature[:] = 1.0
        dt = 1e-5
        vstar = momentum_predict(state, ops, params, dt)
        inter = ns.interior_mask
        npt.assert_allclose(vstar[inter, 1], dt * params.Ra * params.Pr, rtol=1e-12)
        assert np.abs(vstar[inter, 0]).max() <= 1e-9 * dt * params.Ra * params.Pr

    def test_linear_advection_matches_analytic(self, dvd_setup):
        ns, ops, params, _, _ = dvd_setup
        x, y = ns.positions[:, 0], ns.positions[:, 1]
        state = FieldState.zeros(len(ns), 2)
        state.velocity[:, 0] = 1.0 + 2 * x - y
        state.velocity[:, 1] = 0.5 - x + 3 * y
        dt = 1e-6
        vstar = momentum_predict(state, ops, params, dt)
        u, w = state.velocity[:, 0], state.velocity[:, 1]
        inter = ns.interior_mask
        npt.assert_allclose((vstar[:, 0] - u)[inter] / dt, -(2 * u - w)[inter], rtol=2e-6)
        npt.assert_allclose((vstar[:, 1] - w)[inter] / dt, -(-u + 3 * w)[inter], rtol=2e-6)

    def test_bitwise_vs_oracle_on_same_weights(self, dvd_setup):
        """Identical inputs and weights -> the fused kernel equals numpy's expression bit for bit."""
        ns, ops, params, _, _ = dvd_setup
        rng = np.random.default_rng(7)
        v = rng.normal(size=(len(ns), 2))
        T = rng.normal(size=len(ns))
        o = SimpleNamespace(dim=2, lap=ops.lap.matrix, d=[p.matrix for p in ops.partials])
        want = O.momentum(o, v, T, params.Ra, params.Pr, 0.3, 1e-5)
        got = momentum_predict(FieldState(v, np.zeros(len(ns)), T), ops,
                               PhysicsParams(params.Ra, params.Pr, t_ref=0.3), 1e-5)
        npt.assert_array_equal(got, want)


class TestPressureSolve:
    def test_zero_rhs_gives_zero_pressure(self, dvd_setup):
        ns, ops, _, settings, _ = dvd_setup
        assert np.abs(pressure_solve(np.zeros((len(ns), 2)), ops, settings, 1e-5)).max() < 1e-8

    def test_manufactured_solution_second_order(self):
        from scipy.sparse.linalg import splu
        errs = []
        for M in (20, 40):
            ns = nodesets.jittered_box(M, seed=3, jitter=0.2)
            ops = build_operators(ns, {"wall:x-"}, PoissonSolveSettings(), boundary_override=tie_override(ns))
            x, y = ns.positions[:, 0], ns.positions[:, 1]
            exact = np.cos(np.pi * x) * np.cos(np.pi * y)
            n = len(ns)
            rhs = np.empty(n + 1)
            rhs[:n] = -2 * np.pi ** 2 * exact
            rhs[ops.boundary_idx] = 0.0
            rhs[n] = 0.0
            sol = splu(ops.poisson_matrix.tocsc()).solve(rhs)[:n]
            errs.append(np.abs((sol - (exact - exact[ops.gauge]))[ops.interior_idx]).max())
        assert errs[0] < 0.1
        assert errs[1] < errs[0] / 2.5

    def test_residual_contract(self, dvd_setup):
        ns, ops, _, settings, _ = dvd_setup
        vstar = np.random.default_rng(0).normal(size=(len(ns), 2))
        apply_velocity_bc(vstar, ops)
        dt = 1e-5
        p = pressure_solve(vstar, ops, settings, dt)
        n = len(ns)
        rhs = np.empty(n + 1)
        rhs[:n] = (ops.partials[0].matrix @ vstar[:, 0] + ops.partials[1].matrix @ vstar[:, 1]) / dt
        rhs[ops.boundary_idx] = 0.0
        rhs[n] = 0.0
        full = np.concatenate([p, [ops._poisson_lambda]])
        assert np.linalg.norm(rhs - ops.poisson_matrix @ full) / np.linalg.norm(rhs) <= 10 * settings.tol

    def test_matches_direct_solve(self, dvd_setup):
        """LU-preconditioned BiCGStab converges to the direct solution."""
        ns, ops, _, settings, _ = dvd_setup
        vstar = np.random.default_rng(11).normal(size=(len(ns), 2))
        apply_velocity_bc(vstar, ops)
        p = pressure_solve(vstar, ops, settings, 1e-5)
        n = len(ns)
        rhs = np.zeros(n + 1)
        rhs[:n] = (ops.partials[0].matrix @ vstar[:, 0] + ops.partials[1].matrix @ vstar[:, 1]) / 1e-5
        rhs[ops.boundary_idx] = 0.0
        direct = ops.poisson_precond @ rhs
        assert rel(p, direct[:n]) <= 1e-10

    def test_gauge_pinned_to_zero(self, dvd_setup):
        ns, ops, _, settings, _ = dvd_setup
        vstar = np.random.default_rng(1).normal(size=(len(ns), 2))
        apply_velocity_bc(vstar, ops)
        p = pressure_solve(vstar, ops, settings, 1e-5)
        assert abs(p[ops.gauge]) < 1e-10 * np.abs(p).max()


class TestVelocityCorrect:
    def test_constant_pressure_is_identity_inside(self, dvd_setup):
        ns, ops, _, _, _ = dvd_setup
        vstar = np.random.default_rng(2).normal(size=(len(ns), 2))
        apply_velocity_bc(vstar, ops)
        v = velocity_correct(vstar, np.ones(len(ns)), ops, 1e-5)
        npt.assert_allclose(v[ops.interior_idx], vstar[ops.interior_idx], atol=1e-12)

    def test_boundary_is_noslip(self, dvd_setup):
        ns, ops, _, settings, _ = dvd_setup
        vstar = np.random.default_rng(3).normal(size=(len(ns), 2))
        apply_velocity_bc(vstar, ops)
        p = pressure_solve(vstar, ops, settings, 1e-5)
        npt.assert_array_equal(velocity_correct(vstar, p, ops, 1e-5)[ops.boundary_idx], 0.0)

    def test_projection_reduces_divergence_bulk(self, dvd_setup):
        ns, ops, _, settings, _ = dvd_setup
        x, y = ns.positions[:, 0], ns.positions[:, 1]
        bump = (np.sin(np.pi * x) * np.sin(np.pi * y)) ** 4
        vstar = np.stack([bump * np.cos(2 * np.pi * y), bump * np.sin(2 * np.pi * x)], axis=1)
        apply_velocity_bc(vstar, ops)
        before = interior_divergence(vstar, ops)
        v = velocity_correct(vstar, pressure_solve(vstar, ops, settings, 1e-5), ops, 1e-5)
        assert interior_divergence(v, ops) < 0.1 * before

    def test_projection_wall_leak_bounded(self, dvd_setup):
        ns, ops, _, settings, _ = dvd_setup
        x, y = ns.positions[:, 0], ns.positions[:, 1]
        vstar = np.stack([np.sin(np.pi * x) * np.cos(np.pi * y), np.cos(np.pi * x) * np.sin(np.pi * y)], axis=1)
        apply_velocity_bc(vstar, ops)
        before = interior_divergence(vstar, ops)
        v = velocity_correct(vstar, pressure_solve(vstar, ops, settings, 1e-5), ops, 1e-5)
        assert interior_divergence(v, ops) < 0.5 * before


class TestTemperatureStep:
    def test_conduction_profile_is_steady(self, dvd_setup):
        ns, ops, _, _, _ = dvd_setup
        state = FieldState.zeros(len(ns), 2)
        state.temperature = ns.positions[:, 0] - 0.5
        assert np.abs(temperature_step(state, ops, 2e-5) - state.temperature).max() < 1e-9

    def test_insulated_walls_have_zero_normal_gradient(self, dvd_setup):
        ns, ops, _, _, _ = dvd_setup
        state = FieldState.zeros(len(ns), 2)
        state.temperature = np.random.default_rng(4).normal(size=len(ns))
        out = temperature_step(state, ops, 1e-6)
        assert np.abs(ops._w_neumann @ out).max() <= 1e-6 * np.abs(out).max()

    def test_bc_bitwise_vs_oracle(self, dvd_setup):
        ns, ops, _, _, _ = dvd_setup
        T = np.random.default_rng(8).normal(size=len(ns))
        o = SimpleNamespace(dirichlet_idx=ops.dirichlet_idx, dirichlet_values=ops.dirichlet_values,
                            neu_lu=ops.neumann_lu, neumann_idx=ops.neumann_idx, w_neu=ops._w_neumann)
        npt.assert_array_equal(apply_temperature_bc(T.copy(), ops), O.temperature_bc(o, T.copy()))

    def test_heat_decay_rate_second_order(self):
        rates = []
        for M in (20, 40):
            ns = nodesets.regular_box(M)
            ops = build_operators(ns, {"wall:x-"}, PoissonSolveSettings(), boundary_override=tie_override(ns))
            h = 1.0 / M
            state = FieldState.zeros(len(ns), 2)
            state.temperature = np.sin(np.pi * ns.positions[:, 0])
            ops.dirichlet_values = np.zeros(len(ops.dirichlet_idx))
            apply_temperature_bc(state.temperature, ops)
            dt = 0.1 * h * h / 2
            for _ in range(100):
                state.temperature = temperature_step(state, ops, dt)
            probe = ns.interior_mask & (np.abs(np.sin(np.pi * ns.positions[:, 0])) > 0.3)
            ratio = state.temperature[probe] / np.sin(np.pi * ns.positions[probe, 0])
            rates.append(-np.log(np.mean(ratio)) / (100 * dt))
        err = [abs(r - np.pi ** 2) for r in rates]
        assert err[0] < 0.05 * np.pi ** 2
        assert err[1] < err[0] / 2.5


class TestNusselt:
    def test_conduction_limit_is_one(self, dvd_setup):
        ns, ops, _, _, _ = dvd_setup
        state = FieldState.zeros(len(ns), 2)
        state.temperature = ns.positions[:, 0] - 0.5
        assert nusselt_average(state, ops) == pytest.approx(1.0, abs=1e-8)

    def test_constant_temperature_is_zero(self, dvd_setup):
        ns, ops, _, _, _ = dvd_setup
        state = FieldState.zeros(len(ns), 2)
        state.temperature[:] = 0.25
        assert nusselt_average(state, ops) == pytest.approx(0.0, abs=1e-10)


# ---------------------------------------------------------------- parity with the reference's own steps
@pytest.mark.parametrize("case", ["dvd_coarse", "config2_small", "config4_small"])
def test_steps_match_reference_golden(golden, case):
    ns, g = golden(case)
    settings = PoissonSolveSettings()
    ops = build_operators(ns, {"wall:x-"}, settings, boundary_override=tie_override(ns),
                          interior_rbf_n=20 if ns.dim == 3 else None)
    assert ops.gauge == int(g["gauge"])
    dt, Ra, Pr = float(g["dt"]), float(g["Ra"]), float(g["Pr"])
    state = FieldState(np.zeros((len(ns), ns.dim)), np.zeros(len(ns)), g["T0"].copy())
    stepper = DeviceStepper(ops, PhysicsParams(Ra, Pr), settings, dt, state)
    for k in range(int(g["steps"])):
        stepper.step()
        if k == 0:
            s1 = stepper.state()
            for got, ref in ((s1.velocity, g["v1"]), (s1.temperature, g["T1"]), (s1.pressure, g["p1"])):
                assert rel(got, ref) <= FIELD_TOL
    stepper.check_finite(int(g["steps"]))
    sK = stepper.state()
    for got, ref, name in ((sK.velocity, g["vK"], "v"), (sK.temperature, g["TK"], "T"), (sK.pressure, g["pK"], "p")):
        assert rel(got, ref) <= FIELD_TOL, name
    assert stepper.nusselt() == pytest.approx(float(g["nuK"]), rel=1e-8)


def test_hyper_dissipation_steps_match_reference_golden(golden):
    """PhysicsParams.dissipation != 0 (solver.py:235-247): the reference's own 20 steps with the
    fourth-difference term (it moves v by 14 % here, so the path is exercised)."""
    ns, g = golden("dvd_coarse")
    settings = PoissonSolveSettings()
    ops = build_operators(ns, {"wall:x-"}, settings, boundary_override=tie_override(ns))
    dt, Ra, Pr = float(g["hd_dt"]), float(g["hd_Ra"]), float(g["hd_Pr"])
    state = FieldState(np.zeros((len(ns), ns.dim)), np.zeros(len(ns)), g["hd_T0"].copy())
    stepper = DeviceStepper(ops, PhysicsParams(Ra, Pr, dissipation=float(g["hd_dissipation"])), settings, dt, state)
    for _ in range(int(g["hd_steps"])):
        stepper.step()
    sK = stepper.state()
    for got, ref, name in ((sK.velocity, g["hd_vK"], "v"), (sK.temperature, g["hd_TK"], "T"),
                           (sK.pressure, g["hd_pK"], "p")):
        assert rel(got, ref) <= FIELD_TOL, name
    # the standalone API functions take the same path
    st0 = FieldState(np.zeros((len(ns), 2)) + 0.01, np.zeros(len(ns)), g["hd_T0"].copy())
    params = PhysicsParams(Ra, Pr, dissipation=float(g["hd_dissipation"]))
    o = O.build_operators(ns, {"wall:x-"})
    o_mom = O.momentum(o, st0.velocity, st0.temperature, Ra, Pr, 0.0, dt, dissipation=params.dissipation)
    assert rel(momentum_predict(st0, ops, params, dt), o_mom) <= 1e-12
    o_t = O.temperature(o, st0.velocity, st0.temperature.copy(), dt, dissipation=params.dissipation)
    inner = ns.interior_mask  # boundary values come from the tie-row stencils (A5), compared above
    assert rel(temperature_step(st0, ops, dt, params.dissipation)[inner], o_t[inner]) <= 1e-12


def test_stepper_bitwise_deterministic(golden):
    ns, g = golden("dvd_coarse")
    settings = PoissonSolveSettings()
    ops = build_operators(ns, {"wall:x-"}, settings)
    outs = []
    for _ in range(2):
        ops._poisson_lambda = 0.0
        st = DeviceStepper(ops, PhysicsParams(1e6, 0.71), settings, float(g["dt"]),
                           FieldState(np.zeros((len(ns), 2)), np.zeros(len(ns)), g["T0"].copy()))
        for _ in range(5):
            st.step()
        outs.append(st.state())
    assert outs[0].velocity.tobytes() == outs[1].velocity.tobytes()
    assert outs[0].temperature.tobytes() == outs[1].temperature.tobytes()


def test_long_run_parity_vs_oracle():
    """200 steps of config 3's physics on a reduced node set: fields within 1e-8 of the oracle."""
    ns = nodesets.hybrid_hole_2d(40, seed=2)
    settings = PoissonSolveSettings()
    ovr = tie_override(ns)
    ops = build_operators(ns, {"wall:x-"}, settings, boundary_override=ovr)
    o = O.build_operators(ns, {"wall:x-"})
    dt = TimeControls.from_spacing(float(np.min(ns.spacing)), 1.0, Ra=1e6).dt
    T0 = (ns.positions[:, 0] - 0.5) + 1e-3 * np.random.default_rng(0).normal(size=len(ns))
    st = FieldState(np.zeros((len(ns), 2)), np.zeros(len(ns)), T0)
    apply_temperature_bc(st.temperature, ops)
    stepper = DeviceStepper(ops, PhysicsParams(1e6, 0.71), settings, dt, st)
    state, p = (np.zeros((len(ns), 2)), st.temperature.copy()), None
    for _ in range(200):
        stepper.step()
        state, p = O.step(o, state, 1e6, 0.71, 0.0, dt, p_prev=p)
    got = stepper.state()
    assert rel(got.velocity, state[0]) <= FIELD_TOL
    assert rel(got.temperature, state[1]) <= FIELD_TOL
    assert rel(got.pressure, p) <= FIELD_TOL


class TestRun:
    def config(self, **kw):
        base = dict(case="dvd", discretization="hybrid", Ra=1e6, Pr=0.71, t_cold=-0.5, t_hot=0.5, t_init=0.0,
                    t_end=0.002, poisson_tol=1e-8, poisson_maxiter=2000, steady_tol=1e-6, nu_window=40, nu_stride=20,
                    cold_origins={"wall:x-"})
        base.update(kw)
        return SimpleNamespace(**base)

    def test_no_temperature_difference_no_flow(self):
        ns = nodesets.regular_box(20)
        ns.bc_value[ns.role == 1] = 0.2
        res = run(self.config(t_cold=0.2, t_hot=0.2, t_init=0.2), nodeset=ns)
        assert res.final_nu == pytest.approx(0.0, abs=1e-9)
        assert np.abs(res.state.velocity).max() < 1e-9

    def test_bitwise_deterministic_and_bcs(self):
        ns = nodesets.hybrid_hole_2d(30, seed=5)
        a = run(self.config(), nodeset=ns)
        b = run(self.config(), nodeset=ns)
        assert a.nu_values.tobytes() == b.nu_values.tobytes()
        assert a.state.velocity.tobytes() == b.state.velocity.tobytes()
        npt.assert_array_equal(a.state.velocity[ns.boundary_mask], 0.0)
        mask = ns.role == 1
        npt.assert_array_equal(a.state.temperature[mask], ns.bc_value[mask])


@pytest.mark.parametrize("inverse,keep,tol", [(False, 0, 1e-12), (True, 0, 1e-9), (2, 0, 1e-9), (False, 12, 1e-10),
                                              (True, 6, 1e-9), (None, None, 1e-9)])
def test_device_lu_solve_matches_superlu(inverse, keep, tol):
    """The GPU preconditioner (SuperLU factors, supernodal sync-free solves over packed dense
    panels) against SuperLU's own solve: substitution to rounding, diagonal-tile inverses and
    the dense groups (explicit inverses of the top-of-tree row runs; keep = the block levels
    left to the task chain) to the drift DESIGN.md states; twice in a row: bitwise reproducible."""
    from paper_2303_01760_b200 import _lib as L
    from paper_2303_01760_b200.solver import _DeviceLU
    from scipy.sparse import linalg as spla
    ns = nodesets.hybrid_hole_2d(60, seed=2)
    ops = hn.build_operators(ns, {"wall:x-"}, PoissonSolveSettings())
    lu = spla.splu(ops.poisson_matrix.tocsc())  # the factorisation build_operators makes
    dlu = _DeviceLU(lu, inverse=inverse, keep_levels=keep)
    if keep:
        assert dlu.group_rows > 0 and dlu.sL.n_phases >= 1
        assert dlu.sU.group_rows == dlu.sL.group_rows
    elif keep == 0:
        assert dlu.group_rows == 0
    assert int((dlu.sL.w.cpu().numpy() > 32).sum()) > 0  # multi-tile blocks exercised
    b = np.random.default_rng(3).normal(size=dlu.n)
    ref = lu.solve(b)
    t = L.torch()
    bd, xd = L.to_device(b), L.empty(dlu.n, t.float64)
    dlu.solve(bd, xd)
    got = xd.cpu().numpy().copy()
    dlu.solve(bd, xd)
    assert got.tobytes() == xd.cpu().numpy().tobytes()
    assert np.abs(got - ref).max() / np.abs(ref).max() <= tol


@pytest.mark.parametrize("cap,helper", [(32, 64), (96, 512), (256, 4096)])
@pytest.mark.parametrize("inverse,keep", [(False, 0), (True, 0), (2, 0), (False, 5), (True, 20), (2, 60)])
def test_device_lu_random_fill_all_block_shapes(cap, helper, inverse, keep):
    """Random sparse matrix with heavy fill: blocks of every width up to the cap (partial last
    panels, upper and lower), helper-fed blocks and batched small blocks, dense groups cut at
    several depths (many runs and phases), vs SuperLU."""
    from paper_2303_01760_b200 import _lib as L
    from paper_2303_01760_b200.solver import _DeviceLU
    from scipy import sparse
    from scipy.sparse import linalg as spla
    n = 3000
    a = sparse.random(n, n, density=0.004, random_state=7, format="csc") + sparse.eye(n) * 2.0
    lu = spla.splu(a.tocsc())
    dlu = _DeviceLU(lu, inverse=inverse, keep_levels=keep, cap=cap, helper_nnz=helper)
    assert dlu.group_rows == 0 if keep == 0 else (dlu.group_rows > 0 or keep > 20)
    b = np.random.default_rng(5).normal(size=n)
    t = L.torch()
    xd = L.empty(n, t.float64)
    dlu.solve(L.to_device(b), xd)
    ref = lu.solve(b)
    assert np.abs(xd.cpu().numpy() - ref).max() / np.abs(ref).max() <= (1e-9 if inverse or keep else 1e-11)


# ---------------------------------------------------------------- run(): reference loop semantics
def _run_config(g, **over):
    Ra, Pr, t_cold, t_hot, t_init, t_end, stride = (float(v) for v in g["run_cfg"])
    base = dict(case="dvd", discretization="hybrid", Ra=Ra, Pr=Pr, t_cold=t_cold, t_hot=t_hot, t_init=t_init,
                t_end=t_end, poisson_tol=1e-8, poisson_maxiter=2000, steady_tol=1e-6, nu_window=40,
                nu_stride=int(stride), cold_origins={"wall:x-"})
    base.update(over)
    return SimpleNamespace(**base)


def test_run_matches_reference_golden(golden):
    """run() against the reference's own solver.run on a tie-free node set (A22)."""
    ns, g = golden("run_jittered")
    res = run(_run_config(g), nodeset=ns)
    assert res.steps == int(g["run_steps"])
    assert res.dt == pytest.approx(float(g["run_dt"]), rel=0, abs=0)
    npt.assert_array_equal(res.nu_steps, g["run_nu_steps"])
    npt.assert_allclose(res.nu_values, g["run_nu_values"], rtol=1e-8)
    for got, ref in ((res.state.velocity, g["run_v"]), (res.state.temperature, g["run_T"]),
                     (res.state.pressure, g["run_p"])):
        assert rel(got, ref) <= FIELD_TOL
    div = np.asarray(res.diagnostics["divergence_samples"], dtype=float)
    assert div.shape == g["run_div"].shape
    npt.assert_array_equal(div[:, 0], g["run_div"][:, 0])
    npt.assert_allclose(div[:, 1:], g["run_div"][:, 1:], rtol=1e-6)


def test_run_divergence_reports_reference_step_and_node(golden):
    """The finite probe fires at the reference's step with its node (solver.py:448-452),
    although the host reads the device latch only every nu_stride steps."""
    from paper_2303_01760_b200.errors import SolverDivergenceError
    ns, g = golden("run_jittered")
    Pr, t_end = (float(v) for v in g["div_cfg"])
    with pytest.raises(SolverDivergenceError) as exc:
        run(_run_config(g, Pr=Pr, t_end=t_end), nodeset=ns)
    assert exc.value.step == int(g["div_step"])
    assert exc.value.node == int(g["div_node"])


def test_pressure_retry_after_bicgstab_failure(dvd_setup, monkeypatch):
    """A failed BiCGStab is retried by the GMRES stand-in for lgmres (solver.py:306-312), which
    reaches the direct solution; both failing raises PoissonConvergenceError with a residual."""
    from paper_2303_01760_b200 import solver as S
    from paper_2303_01760_b200.errors import PoissonConvergenceError
    ns, ops, _, settings, _ = dvd_setup
    vstar = np.random.default_rng(21).normal(size=(len(ns), 2))
    apply_velocity_bc(vstar, ops)
    n = len(ns)
    rhs = np.zeros(n + 1)
    rhs[:n] = (ops.partials[0].matrix @ vstar[:, 0] + ops.partials[1].matrix @ vstar[:, 1]) / 1e-5
    rhs[ops.boundary_idx] = 0.0
    direct = ops.poisson_precond @ rhs
    orig = S._NativePressure.solve

    def failing(self, b, x0, x, rtol, maxiter, status):  # the device solve reports a breakdown
        orig(self, b, x0, x, rtol, maxiter, status)
        status[0] = -10
        x.zero_()

    monkeypatch.setattr(S._NativePressure, "solve", failing)
    ops._poisson_lambda = 0.0
    p = pressure_solve(vstar, ops, settings, 1e-5)
    assert rel(p, direct[:n]) <= 1e-9
    monkeypatch.setattr(S._GMRES, "solve", lambda self, b, x0, rtol, maxiter: (b.clone(), 7))
    with pytest.raises(PoissonConvergenceError) as exc:
        pressure_solve(vstar, ops, settings, 1e-5)
    assert exc.value.residual > 0


def test_native_pressure_matches_direct_and_scipy_semantics(dvd_setup):
    """hn_pressure_solve (device-driven BiCGStab, graph WHILE node): the direct solution from a
    zero and from a warm start; b = 0 gives x = 0; tol = 0 ends as scipy's does (maxiter or breakdown)."""
    from paper_2303_01760_b200 import _lib as L
    ns, ops, _, settings, _ = dvd_setup
    t = L.torch()
    n1 = ops.n + 1
    b = np.random.default_rng(4).normal(size=n1)
    b[ops.boundary_idx] = 0.0
    b[-1] = 0.0
    direct = ops.poisson_precond @ b
    bd, x, st = L.to_device(b), L.empty(n1, t.float64), L.zeros(2, t.int32)
    ops._d_press.solve(bd, None, x, 1e-8, 2000, st)
    assert st.cpu().numpy()[0] == 0
    assert rel(x.cpu().numpy(), direct) <= 1e-9
    x0 = L.to_device(direct * (1 + 1e-3))
    ops._d_press.solve(bd, x0, x, 1e-8, 2000, st)
    assert st.cpu().numpy()[0] == 0 and rel(x.cpu().numpy(), direct) <= 1e-9
    ops._d_press.solve(bd, x, x, 1e-8, 2000, st)  # warm start from x itself
    assert st.cpu().numpy()[0] == 0 and rel(x.cpu().numpy(), direct) <= 1e-9
    ops._d_press.solve(L.zeros(n1, t.float64), None, x, 1e-8, 2000, st)
    assert st.cpu().numpy()[0] == 0 and not x.cpu().numpy().any()
    # tol = 0 never converges: scipy runs into maxiter or, with the complete-LU preconditioner,
    # into its rho breakdown once the residual is at rounding level; same info here
    from scipy.sparse import linalg as spla
    _, sinfo = spla.bicgstab(ops.poisson_matrix, b, rtol=0.0, atol=0.0, maxiter=3, M=ops.poisson_precond)
    ops._d_press.solve(bd, None, x, 0.0, 3, st)
    info, passes = st.cpu().numpy().tolist()
    assert info != 0 and passes <= 3 and (info == sinfo or {info, sinfo} <= {3, -10, -11})


def test_stepper_rolls_back_and_raises_at_the_failing_step(dvd_setup):
    """tol = 1e-300 makes every BiCGStab (and the retry) fail: the graph-mode stepper latches the
    failure on the device, and check_finite rolls back, replays step 1 with the reference's
    handling and raises PoissonConvergenceError there (solver.py:304-313)."""
    from paper_2303_01760_b200.errors import PoissonConvergenceError
    ns, ops, params, _, _ = dvd_setup
    st = FieldState(np.zeros((len(ns), 2)), np.zeros(len(ns)), (ns.positions[:, 0] - 0.5).copy())
    apply_temperature_bc(st.temperature, ops)
    stepper = DeviceStepper(ops, params, PoissonSolveSettings(tol=1e-300, maxiter=2), 1e-5, st)
    for _ in range(4):
        stepper.step()
    with pytest.raises(PoissonConvergenceError):
        stepper.check_finite()
    assert stepper.steps == 0  # rolled back to the start, failed again at step 1


def test_run_generates_its_node_set_on_the_device():
    """run(CaseConfig) with no nodeset: domain, device node generation, operators and the loop
    (reference solver.py:412-419); the same call with the generated set passed in is bitwise equal."""
    import paper_2303_01760_b200 as hn
    cfg = hn.CaseConfig(case="dvd", h_r=0.05, t_end=2e-4)
    a = run(cfg)
    ns = hn.hybrid_discretize(cfg)
    assert len(a.nodeset) == len(ns) and np.array_equal(a.nodeset.positions, ns.positions)
    b = run(cfg, nodeset=ns)
    assert a.steps == b.steps >= 1
    assert a.state.temperature.tobytes() == b.state.temperature.tobytes()
    assert np.isfinite(a.final_nu)


def test_run_obstacle_case_with_precomputed_node_set():
    """CaseConfig.cold_origins(spec) reads spec.obstacles: run() builds the domain even when
    the node set is given (reference solver.py:412-415)."""
    import paper_2303_01760_b200 as hn
    cfg = hn.CaseConfig(case="obstacles2d", h_r=0.04, t_end=1e-4)
    ns = hn.hybrid_discretize(cfg)
    res = run(cfg, nodeset=ns)
    assert res.steps >= 1 and np.isfinite(res.final_nu)
    assert np.isfinite(res.state.velocity).all()


def test_pressure_solve_runs_several_passes_with_an_inexact_preconditioner():
    """The device BiCGStab beyond its first half-step: the factors of A precondition a slightly
    perturbed matrix, so the WHILE node iterates and the IF node around a pass's second half is
    entered; same pass count as scipy's bicgstab, solution at the direct solve of the perturbed
    system."""
    from scipy.sparse import linalg as spla

    from paper_2303_01760_b200 import _lib as L
    from paper_2303_01760_b200.operators import DeviceCSR
    from paper_2303_01760_b200.solver import _NativePressure
    ns = nodesets.hybrid_hole_2d(40, seed=5)
    ops = hn.build_operators(ns, {"wall:x-"}, PoissonSolveSettings())
    A = ops.poisson_matrix.tocsr()
    rng = np.random.default_rng(1)
    A2 = A.copy()
    A2.data = A2.data * (1.0 + 1e-5 * rng.normal(size=A2.nnz))
    b = rng.normal(size=A.shape[0])
    lu = spla.splu(A.tocsc())
    count = [0]

    def cb(_):
        count[0] += 1

    xs, sinfo = spla.bicgstab(A2, b, rtol=1e-12, atol=0.0, maxiter=200, M=spla.LinearOperator(A.shape, lu.solve),
                              callback=cb)
    assert sinfo == 0 and count[0] >= 2, (sinfo, count[0])
    t = L.torch()
    press = _NativePressure(DeviceCSR(A2), ops._d_lu)
    x = L.empty(A.shape[0], t.float64)
    status = L.zeros(2, t.int32)
    press.solve(L.to_device(b), None, x, 1e-12, 200, status)
    info, passes = (int(v) for v in status.cpu().numpy())
    assert info == 0 and abs(passes - count[0]) <= 1, (info, passes, count[0])
    ref = spla.spsolve(A2.tocsc(), b)
    scale = np.abs(ref).max()
    assert np.abs(x.cpu().numpy() - ref).max() / scale <= 10 * max(np.abs(xs - ref).max() / scale, 1e-9)
