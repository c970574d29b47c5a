"""Host-side logic that needs no GPU: triangular-solve task planning (emulated task by
task in ticket order, the order the kernel's atomic ticket hands them out), node-set
generators, operator-code mapping."""

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

from paper_2303_01760_b200 import nodesets
from paper_2303_01760_b200.approx import _op_code, Laplacian, NormalDerivative, Partial
from paper_2303_01760_b200.solver import plan_triangular_tasks


def emulate(plan, m, b, diag=None):
    """Execute the task list sequentially in ticket order (a valid schedule)."""
    x = np.full(m.shape[0], np.nan)
    partial = np.full(max(plan["npartial"], 1), np.nan)
    for t in range(plan["ntasks"]):
        r, e0, ln = plan["row"][t], plan["beg"][t], plan["len"][t]
        cols = m.indices[e0:e0 + ln]
        assert not np.any(np.isnan(x[cols])), "task ran before a dependency"
        s = float(np.dot(m.data[e0:e0 + ln], x[cols]))
        if plan["np"][t] < 0:
            partial[plan["part"][t]] = s
        else:
            p0, k = plan["part"][t], plan["np"][t]
            assert not np.any(np.isnan(partial[p0:p0 + k]))
            tot = float(np.sum(partial[p0:p0 + k])) + s
            x[r] = (b[r] - tot) / (diag[r] if diag is not None else 1.0)
    return x


@pytest.mark.parametrize("lower", [True, False])
@pytest.mark.parametrize("chunk", [4, 256])
def test_task_plan_solves_triangular_systems(lower, chunk):
    rng = np.random.default_rng(0)
    n = 400
    a = sp.random(n, n, density=0.05, random_state=1, format="csr")
    a = a + sp.csr_matrix((np.ones(n), (np.full(n, n - 1 if lower else 0), np.arange(n))), shape=(n, n))
    tri = sp.tril(a, k=-1, format="csr") if lower else sp.triu(a, k=1, format="csr")
    tri.sort_indices()
    b = rng.normal(size=n)
    diag = rng.uniform(1, 2, size=n)
    plan = plan_triangular_tasks(tri, lower, chunk)
    x = emulate(plan, tri, b, None if lower else diag)
    full = (tri + sp.eye(n)) if lower else (tri + sp.diags(diag))
    want = spsolve_triangular(full.tocsr(), b, lower=lower)
    np.testing.assert_allclose(x, want, rtol=1e-10, atol=1e-12)
    assert plan["ntasks"] >= n
    if chunk == 4:
        assert plan["npartial"] > 0


def test_generators_match_baseline_sizes():
    assert len(nodesets.regular_box(199)) == 40_000
    ns = nodesets.jittered_box(315, seed=1)
    assert len(ns) == 99_856 and ns.counts == (0, 98_596, 1_260)
    ns = nodesets.hybrid_hole_2d(500, seed=2)
    assert 240_000 < len(ns) < 255_000 and 0.2 < ns.counts[1] / len(ns) < 0.26


def test_generator_lattice_map_is_consistent():
    ns = nodesets.hybrid_hole_2d(40, seed=3)
    grid = ns.lattice.grid
    ids = grid[grid >= 0]
    keys = ns.lattice_idx[ids]
    np.testing.assert_array_equal(grid[keys[:, 0], keys[:, 1]], ids)
    np.testing.assert_allclose(ns.positions[ids], keys * ns.lattice.step, atol=1e-15)


def test_config0_generator_matches_reference_generator():
    """regular_box(199) is the reference's dvd pure-regular set (counts, roles, lattice)."""
    import sys
    from pathlib import Path
    ref = Path("/root/reference/pkg/src")
    if not ref.exists():
        pytest.skip("reference not mounted (GPU box)")
    sys.path.insert(0, str(ref))
    from hybridnodes.config import CaseConfig
    from hybridnodes.nodegen import hybrid_discretize
    r = hybrid_discretize(CaseConfig(case="dvd", discretization="pure-regular", h_r=1 / 49))
    ours = nodesets.regular_box(49)
    assert r.counts == ours.counts
    np.testing.assert_allclose(np.sort(r.positions, axis=0), np.sort(ours.positions, axis=0), atol=1e-14)
    assert sorted(r.origin) == sorted(ours.origin)
    assert (r.role == 1).sum() == (ours.role == 1).sum()


def test_operator_codes_accept_foreign_operator_classes():
    class Laplacian_:  # a class from another package with the same name
        pass
    Laplacian_.__name__ = "Laplacian"
    assert _op_code(Laplacian(), 2)[0] == 0
    assert _op_code(Laplacian_(), 2)[0] == 0
    assert _op_code(Partial(1), 3) == (1, 1, (0.0, 0.0, 0.0))
    assert _op_code(NormalDerivative((0.6, 0.8)), 2) == (2, 0, (0.6, 0.8))
    with pytest.raises(TypeError):
        _op_code(object(), 2)


def emulate_blocks(plan, m, b, lower, diag=None):
    """Execute the supernodal task list sequentially in ticket order (helpers included)."""
    n = m.shape[0]
    x = np.full(n, np.nan)
    ysum = np.full(n, np.nan)
    dense = m.toarray()

    def outside(i, r0, w):
        c = m.indices[m.indptr[i]:m.indptr[i + 1]]
        v = m.data[m.indptr[i]:m.indptr[i + 1]]
        out = (c < r0) if lower else (c >= r0 + w)
        assert not np.any(np.isnan(x[c[out]])), "task ran before a dependency"
        assert np.array_equal(np.sort(c[~out]), np.arange(r0, i) if lower else np.arange(i + 1, r0 + w))
        return b[i] - np.dot(v[out], x[c[out]])

    nt = plan["ntasks"]
    for kind, r0, w, rb, rc in zip(plan["kind"][:nt], plan["t_r0"][:nt], plan["t_w"][:nt], plan["t_rb"][:nt],
                                   plan["t_rc"][:nt]):
        rows = np.arange(r0, r0 + w)
        if kind == 3:  # batch: members run concurrently -> all outside sums before any solve
            mem = [(plan["t_r0"][k], plan["t_w"][k]) for k in range(rb, rb + rc)]
            assert all(plan["kind"][k] == 4 for k in range(rb, rb + rc)) and all(mw <= 32 for _, mw in mem)
            ys = [np.array([outside(i, mr0, mw) for i in range(mr0, mr0 + mw)]) for mr0, mw in mem]
            for (mr0, mw), y in zip(mem, ys):
                mrows = np.arange(mr0, mr0 + mw)
                blk = dense[np.ix_(mrows, mrows)]
                full = blk + (np.eye(mw) if lower else np.diag(diag[mrows]))
                x[mrows] = spsolve_triangular(sp.csr_matrix(full), y, lower=lower)
            continue
        if kind == 1:
            for i in range(r0 + rb, r0 + rb + rc):
                ysum[i] = outside(i, r0, w)
            continue
        if kind == 2:
            assert not np.any(np.isnan(ysum[rows])), "dense part before its helpers"
            y = ysum[rows].copy()
        else:
            y = np.array([outside(i, r0, w) for i in rows])
        blk = dense[np.ix_(rows, rows)]
        full = blk + (np.eye(w) if lower else np.diag(diag[rows]))
        x[rows] = spsolve_triangular(sp.csr_matrix(full), y, lower=lower)
    return x


@pytest.mark.parametrize("lower", [True, False])
def test_supernodal_plan_solves_triangular_systems(lower):
    from paper_2303_01760_b200.solver import plan_supernodal_blocks
    from scipy.sparse import linalg as spla
    rng = np.random.default_rng(1)
    n = 300
    a = sp.random(n, n, density=0.03, random_state=2, format="csc") + sp.eye(n) * 4
    lu = spla.splu(a.tocsc())
    tri = sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr") if lower else sp.triu(sp.csr_matrix(lu.U), k=1, format="csr")
    tri.sort_indices()
    diag = sp.csr_matrix(lu.U).diagonal()
    plan = plan_supernodal_blocks(tri, lower, cap=64, helper_nnz=40)
    assert plan["nblk"] < n and plan["w"].sum() == n
    assert plan["heavy"] > 0 and plan["batched"] > 0
    b = rng.normal(size=n)
    x = emulate_blocks(plan, tri, b, lower, diag)
    full = (tri + sp.eye(n)) if lower else (tri + sp.diags(diag))
    np.testing.assert_allclose(x, spsolve_triangular(full.tocsr(), b, lower=lower), rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("lower", [True, False])
def test_host_tile_inverse_inverts_every_diagonal_tile(lower):
    """hn_host_tile_inverse (host code, no GPU): row i of tinv is row (i - tile start) of the
    inverse of its 32-row diagonal tile (unit lower / diag-upper), tiles from each block start."""
    from scipy.sparse import linalg as spla

    from paper_2303_01760_b200 import _lib as L
    from paper_2303_01760_b200.solver import plan_supernodal_blocks
    n = 400
    a = sp.random(n, n, density=0.02, random_state=5, format="csc") + sp.eye(n) * 3
    lu = spla.splu(a.tocsc(), permc_spec="NATURAL", diag_pivot_thresh=0.0)
    tri = sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr") if lower else sp.triu(sp.csr_matrix(lu.U), k=1, format="csr")
    tri.sort_indices()
    diag = np.ascontiguousarray(sp.csr_matrix(lu.U).diagonal(), dtype=np.float64)
    plan = plan_supernodal_blocks(tri, lower, cap=96)
    r0, w = np.ascontiguousarray(plan["r0"], np.int32), np.ascontiguousarray(plan["w"], np.int32)
    rowptr = np.ascontiguousarray(tri.indptr, np.int64)
    cols = np.ascontiguousarray(tri.indices, np.int32)
    vals = np.ascontiguousarray(tri.data, np.float64)
    tinv = np.empty(n * 32)
    vp = L._vp
    L.call("hn_host_tile_inverse", rowptr.ctypes.data_as(vp), cols.ctypes.data_as(vp), vals.ctypes.data_as(vp),
           diag.ctypes.data_as(vp), n, 1 if lower else 0, len(r0), r0.ctypes.data_as(vp), w.ctypes.data_as(vp),
           tinv.ctypes.data_as(vp))
    tinv = tinv.reshape(n, 32)
    dense = tri.toarray()
    checked = 0
    for b0, bw in zip(r0, w):
        for t0 in range(0, bw, 32):
            tw = min(32, bw - t0)
            s = slice(b0 + t0, b0 + t0 + tw)
            T = dense[s, s] + (np.eye(tw) if lower else np.diag(diag[s]))
            np.testing.assert_allclose(tinv[s, :tw] @ T, np.eye(tw), atol=1e-10)
            checked += 1
    assert checked > 10


def test_run_builds_the_domain_spec_for_cold_origins(monkeypatch):
    """run(config, nodeset=...) builds the reference's domain spec before cold_origins(spec)
    (reference solver.py:412-415) when the reference config module is importable: obstacle
    cases read spec.obstacles there."""
    import sys
    import types
    from paper_2303_01760_b200 import solver as S

    spec_obj = object()
    fake_cfg = types.ModuleType("hybridnodes.config")
    fake_cfg.build_domain = lambda config: spec_obj
    fake_pkg = types.ModuleType("hybridnodes")
    fake_pkg.config = fake_cfg
    monkeypatch.setitem(sys.modules, "hybridnodes", fake_pkg)
    monkeypatch.setitem(sys.modules, "hybridnodes.config", fake_cfg)

    class Reached(Exception):
        pass

    seen = {}

    class Cfg:
        poisson_tol, poisson_maxiter = 1e-8, 2000

        def cold_origins(self, spec):
            seen["spec"] = spec
            raise Reached

    with pytest.raises(Reached):
        S.run(Cfg(), nodeset=nodesets.jittered_box(8, seed=0))
    assert seen["spec"] is spec_obj
