"""Pin the CPU oracle (oracle/hn_oracle.py) to golden vectors produced by running the
reference itself (oracle/make_golden.py).  Integer outputs and CSR application are
bit-exact; weights agree to LAPACK rounding (the reference's OpenBLAS kernels are
CPU-model dependent) and are bit-exact on the host that made the goldens."""

import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_CASES
from oracle import hn_oracle as O

OPS2 = [("lap",), ("d", 0), ("d", 1)]
OPS3 = [("lap",), ("d", 0), ("d", 1), ("d", 2)]
NAMES = ["lap", "d0", "d1", "d2"]


def rowwise_rel(a, b):
    den = np.maximum(np.abs(b).max(axis=1), 1e-300)
    return (np.abs(a - b).max(axis=1) / den).max()


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_oracle_weights_match_reference(golden, case):
    ns, g = golden(case)
    dim = ns.dim
    ops = OPS2 if dim == 2 else OPS3
    t = O.compute_weights(ns, ops, rbf_n=20 if dim == 3 else None)
    np.testing.assert_array_equal(t["method"], g["method"])
    np.testing.assert_array_equal(t["sizes"], g["sizes"])
    np.testing.assert_array_equal(t["indices"], g["indices"])
    for op, name in zip(ops, NAMES):
        assert rowwise_rel(t["weights"][op], g[f"w_{name}"]) <= 1e-12


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_oracle_apply_bitwise_on_reference_weights(golden, case):
    ns, g = golden(case)
    n = len(ns)
    table = {"indices": g["indices"], "sizes": g["sizes"], "weights": {}}
    for name in NAMES[: ns.dim + 1]:
        table["weights"][name] = g[f"w_{name}"]
        m = O.csr(table, name, n)
        got = O.apply(m, g["field"])
        np.testing.assert_array_equal(got, g[f"apply_{name}"])


def test_oracle_sequential_loop_equals_csr_matvec(golden):
    ns, g = golden("dvd_coarse")
    table = {"indices": g["indices"], "sizes": g["sizes"], "weights": {"lap": g["w_lap"]}}
    m = O.csr(table, "lap", len(ns))
    np.testing.assert_array_equal(O.apply_sequential(m, g["field"]), O.apply(m, g["field"]))


@pytest.mark.parametrize("case", ["dvd_coarse", "config0_small", "config1_small", "config2_small", "config4_small"])
def test_oracle_boundary_tables(golden, case):
    ns, g = golden(case)
    bidx = np.nonzero(ns.boundary_mask)[0]
    bg = O.boundary_table(ns, bidx, ns.boundary_mask)
    np.testing.assert_array_equal(bg["sizes"], g["bgrad_sizes"])
    np.testing.assert_array_equal(bg["indices"], g["bgrad_indices"])
    for a in range(ns.dim):
        assert rowwise_rel(bg["weights"][("d", a)], g[f"bgrad_w_d{a}"]) <= 1e-12
    if "nu_rows" in g:
        nt = O.boundary_table(ns, g["nu_rows"], None, normals=True)
        np.testing.assert_array_equal(nt["indices"], g["nu_indices"])
        assert rowwise_rel(nt["weights"]["normal"], g["nu_w"]) <= 1e-12


@pytest.mark.parametrize("case", ["dvd_coarse", "config2_small", "config4_small"])
def test_oracle_steps_match_reference(golden, case):
    ns, g = golden(case)
    o = O.build_operators(ns, {"wall:x-"}, rbf_n=20 if ns.dim == 3 else None)
    assert o.gauge == int(g["gauge"])
    np.testing.assert_array_equal(o.poisson.indptr, g["poisson_indptr"])
    np.testing.assert_array_equal(o.poisson.indices, g["poisson_indices"])
    np.testing.assert_allclose(o.poisson.data, g["poisson_data"], rtol=1e-11, atol=1e-11 * np.abs(g["poisson_data"]).max())
    dt, Ra, Pr = float(g["dt"]), float(g["Ra"]), float(g["Pr"])
    state = (np.zeros((len(ns), ns.dim)), g["T0"].copy())
    vst = O.momentum(o, state[0], state[1], Ra, Pr, 0.0, dt)
    np.testing.assert_array_equal(vst, g["vstar1_raw"])
    p = None
    for k in range(int(g["steps"])):
        state, p = O.step(o, state, Ra, Pr, 0.0, dt, p_prev=p)
        if k == 0:
            for got, ref in ((state[0], g["v1"]), (state[1], g["T1"]), (p, g["p1"])):
                np.testing.assert_allclose(got, ref, rtol=0, atol=1e-10 * max(np.abs(ref).max(), 1e-300))
    for got, ref in ((state[0], g["vK"]), (state[1], g["TK"]), (p, g["pK"])):
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-8 * max(np.abs(ref).max(), 1e-300))
    assert O.nusselt(o, state[1]) == pytest.approx(float(g["nuK"]), rel=1e-8)


def test_oracle_hyper_dissipation_steps_match_reference(golden):
    """The oracle's dissipation term (solver.py:235-247) against the reference's own steps."""
    ns, g = golden("dvd_coarse")
    o = O.build_operators(ns, {"wall:x-"})
    dt, Ra, Pr, diss = float(g["hd_dt"]), float(g["hd_Ra"]), float(g["hd_Pr"]), float(g["hd_dissipation"])
    state, p = (np.zeros((len(ns), ns.dim)), g["hd_T0"].copy()), None
    for _ in range(int(g["hd_steps"])):
        state, p = O.step(o, state, Ra, Pr, 0.0, dt, p_prev=p, dissipation=diss)
    for got, ref in ((state[0], g["hd_vK"]), (state[1], g["hd_TK"]), (p, g["hd_pK"])):
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-8 * max(np.abs(ref).max(), 1e-300))


def test_oracle_knn_brute_force_tie_order():
    """kNN key = (fl-distance, index), as the reference's own brute-force oracle
    (pkg/tests/test_approx.py:70-83)."""
    rng = np.random.default_rng(5)
    pts = rng.uniform(0, 1, (100, 2))
    got = O.knn_by_key(pts, pts[[0, 17, 63, 99]], 12)
    for row, c in zip(got, (0, 17, 63, 99)):
        d = np.linalg.norm(pts - pts[c], axis=1)
        assert list(row) == sorted(range(100), key=lambda i: (d[i], i))[:12]
    lat = np.array([[i * 0.1, j * 0.1] for i in range(5) for j in range(5)])
    np.testing.assert_array_equal(O.knn_by_key(lat, lat[[12]], 5)[0], [12, 7, 11, 13, 17])


def test_oracle_classic_fd():
    h = 0.1
    lat = np.array([[i * h, j * h] for i in range(5) for j in range(5)])
    st = np.array([[12, 7, 11, 13, 17]])
    w = O.mon_solve(lat, st, [("lap",), ("d", 0)])[0]
    np.testing.assert_allclose(w[:, 0], [-4 / h ** 2, 1 / h ** 2, 1 / h ** 2, 1 / h ** 2, 1 / h ** 2], rtol=1e-12)
    np.testing.assert_allclose(w[[1, 4], 1], [-1 / (2 * h), 1 / (2 * h)], rtol=1e-12)


@pytest.mark.parametrize("case", ["dvd_coarse", "config1_small", "config2_small", "config4_small"])
def test_host_kappa_matches_reference_golden(golden, case):
    """The host restatement of the with_kappa diagnostic (approx._kappa_host, numpy SVD of the
    local systems) against the reference's own compute_weights(with_kappa=True) output
    (tests/golden/kappa_*.npz, oracle/make_golden_kappa.py)."""
    from paper_2303_01760_b200.approx import _kappa_host
    ns, g = golden(case)
    pre = "n30_" if case == "config4_small" else ""
    idx, sizes, method = g[pre + "indices"], g[pre + "sizes"], g[pre + "method"]
    with np.load(GOLDEN / f"kappa_{case}.npz") as z:
        want = z["kappa"]
    got = np.full(len(ns), np.nan)
    for mon in (True, False):
        rows = np.nonzero((sizes > 0) & ((method == 0) == mon))[0]
        if not len(rows):
            continue
        w = int(sizes[rows[0]])
        st = np.array([np.concatenate([[r], [j for j in idx[r, :w] if j != r]]) for r in rows])
        got[rows] = _kappa_host(ns.positions, st, mon)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    fin = np.isfinite(want)
    np.testing.assert_allclose(got[fin], want[fin], rtol=1e-10)
