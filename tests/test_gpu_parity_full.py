"""Field parity at the BASELINE sizes.

* config 3 at full N (hybrid hole set, N = 243,955): build_operators + DeviceStepper against
  the oracle's run-loop body (reference solver.py:439-452) for 50 steps, and for 1,000 steps
  under HN_SLOW=1 (slow marker; the oracle alone needs ~6 min of CPU for it);
* the full-N preconditioner: the device LU solve against SuperLU's own solve;
* the config-4 twin the bench steps (3D sphere set, N = 20,055, interior n = 30): 200 steps;
* the exact-tie boundary rows of SURVEY §8(a) A5 at configs 3 and 4: how many there are and
  how far the fields move when the GPU keeps its own (distance, index) choice.

Tolerance: fields <= 1e-8 relative (max-norm over the field), as the north star states.  The
measured maxima are printed and, with HN_PARITY_REPORT=<path>, written as JSON.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import paper_2303_01760_b200 as hn
from oracle import hn_oracle as O
from paper_2303_01760_b200 import nodesets
from paper_2303_01760_b200.operators import FieldState
from paper_2303_01760_b200.solver import DeviceStepper, PhysicsParams, PoissonSolveSettings, TimeControls

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-8
REPORT: dict = {}


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def record(key, value):
    REPORT[key] = value
    print(f"[parity] {key}: {value}")
    path = os.environ.get("HN_PARITY_REPORT")
    if path:
        old = json.loads(open(path).read()) if os.path.exists(path) else {}
        old.update({key: value})
        with open(path, "w") as f:
            json.dump(old, f, indent=1)


def tie_override(ns, size):
    bidx = np.nonzero(ns.boundary_mask)[0]
    t = hn.boundary_partial_table(ns, bidx, exclude=ns.boundary_mask)
    rows = np.asarray(t.tie_rows, dtype=np.int64)
    st = O.boundary_stencils(ns, rows, ns.boundary_mask, size) if len(rows) else np.empty((0, size))
    return rows, st


def initial_temperature(ns, seed):
    """Config 3/4 initial state: T = (x - 0.5) + 1e-3 N(0,1), seeded."""
    return (ns.positions[:, 0] - 0.5) + 1e-3 * np.random.default_rng(seed).normal(size=len(ns))


class Case:
    def __init__(self, ns, Ra, rbf_n=None, override=True, seed=3):
        self.ns, self.Ra = ns, Ra
        self.rbf_n = rbf_n
        size = hn.RBF_SIZE[ns.dim]
        self.override = tie_override(ns, size) if override else None
        self.ops = hn.build_operators(ns, {"wall:x-"}, PoissonSolveSettings(), boundary_override=self.override,
                                      interior_rbf_n=rbf_n)
        self.dt = TimeControls.from_spacing(float(np.min(ns.spacing)), 1.0, Ra=Ra).dt
        self.T0 = initial_temperature(ns, seed)

    def stepper(self):
        st = FieldState(np.zeros((len(self.ns), self.ns.dim)), np.zeros(len(self.ns)), self.T0.copy())
        hn.apply_temperature_bc(st.temperature, self.ops)
        return DeviceStepper(self.ops, PhysicsParams(self.Ra, 0.71), PoissonSolveSettings(), self.dt, st)


class OracleRun:
    """The reference loop body on the CPU oracle, advanced lazily to any step count."""

    def __init__(self, ns, Ra, T0, rbf_n=None):
        self.o = O.build_operators(ns, {"wall:x-"}, rbf_n=rbf_n)
        self.Ra = Ra
        self.dt = O.dt_rule(float(np.min(ns.spacing)), Ra)
        T = O.temperature_bc(self.o, T0.copy())
        self.state, self.p, self.k = (np.zeros((len(ns), ns.dim)), T), None, 0
        self.snap = {}

    SNAP = (1, 10, 50, 100, 200, 250, 500, 1000)

    def advance_to(self, k):
        if k <= self.k:
            return self.snap[k]
        while self.k < k:
            self.state, self.p = O.step(self.o, self.state, self.Ra, 0.71, 0.0, self.dt, p_prev=self.p)
            self.k += 1
            if self.k in self.SNAP:
                self.snap[self.k] = (self.state, self.p)
        return self.state, self.p


def compare(stepper, orun, k, label):
    (v, T), p = orun.advance_to(k)
    s = stepper.state()
    errs = {"v": rel(s.velocity, v), "T": rel(s.temperature, T), "p": rel(s.pressure, p)}
    record(f"{label}_step{k}", {f: float(f"{e:.3e}") for f, e in errs.items()})
    for f, e in errs.items():
        assert e <= FIELD_TOL, f"{label}: {f} after {k} steps differs by {e:.2e}"
    return errs


# ---------------------------------------------------------------- config 3 at full N
@pytest.fixture(scope="module")
def config3():
    ns = nodesets.hybrid_hole_2d(500, seed=2)
    assert len(ns) == 243955
    case = Case(ns, 1e6)
    orun = OracleRun(ns, 1e6, case.T0)
    assert case.ops.gauge == orun.o.gauge
    return case, orun


def test_config3_full_n_fields_50_steps(config3):
    case, orun = config3
    st = case.stepper()
    for k in (1, 10, 50):
        while st.steps < k:
            st.step()
        compare(st, orun, k, "config3_fullN")
    st.check_finite()


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("HN_SLOW"), reason="1,000 oracle steps take ~6 min of CPU: HN_SLOW=1")
def test_config3_full_n_fields_1000_steps(config3):
    case, orun = config3
    st = case.stepper()
    for k in (100, 250, 500, 1000):
        while st.steps < k:
            st.step()
        compare(st, orun, k, "config3_fullN")
    st.check_finite()


def test_config3_full_n_preconditioner_matches_superlu(config3):
    """The device LU solve (full-N supernodal factors, all helper/batched task kinds) against
    SuperLU's solve of the same factorisation (reference solver.py:213-214)."""
    from paper_2303_01760_b200 import _lib as L
    case, _ = config3
    ops = case.ops
    lu = ops.poisson_precond  # LinearOperator over SuperLU.solve (what the reference applies)
    t = L.torch()
    n1 = ops.n + 1
    worst = 0.0
    for seed in (0, 1):
        b = np.random.default_rng(seed).normal(size=n1)
        ref = lu @ b
        x = L.empty(n1, t.float64)
        ops._d_lu.solve(L.to_device(b), x)
        worst = max(worst, rel(x.cpu().numpy(), ref))
    record("config3_fullN_precond_vs_superlu", float(f"{worst:.3e}"))
    assert worst <= ops._d_lu.parity_tol


def test_config3_tie_rows_own_choice_delta(config3):
    """A5: the GPU's own (distance, index) choice on the exact-tie boundary rows, stepped 10
    times, against the oracle (which keeps the reference's cKDTree choice)."""
    case, orun = config3
    rows = case.override[0]
    own = Case(case.ns, 1e6, override=False)
    st = own.stepper()
    for _ in range(10):
        st.step()
    (v, T), p = orun.advance_to(10)
    s = st.state()
    record("config3_tie_rows", {"count": int(len(rows)), "rows": [int(r) for r in rows[:16]],
                                "own_choice_delta_step10": {"v": float(f"{rel(s.velocity, v):.3e}"),
                                                            "T": float(f"{rel(s.temperature, T):.3e}"),
                                                            "p": float(f"{rel(s.pressure, p):.3e}")}})
    if len(rows) == 0:
        assert rel(s.velocity, v) <= FIELD_TOL


# ---------------------------------------------------------------- config 4 twin (the stepped 3D set)
@pytest.fixture(scope="module")
def config4_twin():
    ns = nodesets.hybrid_sphere_3d(24, seed=4, refine=2.8)
    assert len(ns) == 20055
    case = Case(ns, 1e5, rbf_n=30)
    orun = OracleRun(ns, 1e5, case.T0, rbf_n=30)
    return case, orun


def test_config4_twin_fields_200_steps(config4_twin):
    case, orun = config4_twin
    st = case.stepper()
    for k in (1, 10, 50, 200):
        while st.steps < k:
            st.step()
        compare(st, orun, k, "config4_twin")
    st.check_finite()


def test_config4_twin_tie_rows_own_choice_delta(config4_twin):
    case, orun = config4_twin
    rows = case.override[0]
    own = Case(case.ns, 1e5, rbf_n=30, override=False)
    st = own.stepper()
    for _ in range(10):
        st.step()
    (v, T), p = orun.advance_to(10)
    s = st.state()
    record("config4_twin_tie_rows", {"count": int(len(rows)),
                                     "own_choice_delta_step10": {"v": float(f"{rel(s.velocity, v):.3e}"),
                                                                 "T": float(f"{rel(s.temperature, T):.3e}"),
                                                                 "p": float(f"{rel(s.pressure, p):.3e}")}})
