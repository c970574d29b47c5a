"""Host-side logic that needs no GPU: supernodal triangular-solve planning (emulated task
by task in ticket order, the order the kernel's atomic ticket hands them out) and the
packed dense panels, node-set generators, operator-code mapping."""

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

from paper_2303_01760_b200 import nodesets
from paper_2303_01760_b200.approx import _op_code, Laplacian, NormalDerivative, Partial


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


def _panel_geom(lower, w, tt):
    """Python restatement of panel_geom (csrc/pressure.cu)."""
    ntiles = (w + 31) // 32
    t0 = 32 * tt if lower else 32 * (ntiles - 1 - tt)
    tw = min(32, w - t0)
    rbase = t0 if lower else 0
    rows = w - t0 if lower else t0 + tw
    return t0, tw, rbase, rows, (rows + 1) & ~1


@pytest.mark.parametrize("lower", [True, False])
@pytest.mark.parametrize("cap", [96, 40])
def test_host_pack_panels_hold_every_dense_block(lower, cap):
    """hn_host_pack_panels (host code, no GPU): reading the packed panels back with the
    kernel's geometry gives exactly the strict in-block triangle of every block task and, for
    tasks with a predecessor rectangle (t_rw > 0), the block rows x predecessor columns."""
    from scipy.sparse import linalg as spla

    from paper_2303_01760_b200 import _lib as L
    from paper_2303_01760_b200.solver import plan_supernodal_blocks
    n = 600
    a = sp.random(n, n, density=0.02, random_state=5, format="csc") + sp.eye(n) * 3
    lu = spla.splu(a.tocsc())
    tri = sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr") if lower else sp.triu(sp.csr_matrix(lu.U), k=1, format="csr")
    tri.sort_indices()
    plan = plan_supernodal_blocks(tri, lower, cap=cap, helper_nnz=200)
    kind, r0, w, rw = plan["kind"], plan["t_r0"], plan["t_w"], plan["t_rw"]
    if cap == 40:
        assert plan["rects"] > 0  # supernodes wider than the cap come in dense-coupled pieces
    rowptr = np.ascontiguousarray(tri.indptr, np.int64)
    cols = np.ascontiguousarray(tri.indices, np.int32)
    vals = np.ascontiguousarray(tri.data, np.float64)
    off = np.empty(len(kind), np.int64)
    vp = L._vp
    one = np.ones(1)
    args = (rowptr.ctypes.data_as(vp), cols.ctypes.data_as(vp), vals.ctypes.data_as(vp), one.ctypes.data_as(vp),
            1 if lower else 0, 0, plan["ntasks"], kind.ctypes.data_as(vp), r0.ctypes.data_as(vp),
            w.ctypes.data_as(vp), rw.ctypes.data_as(vp), off.ctypes.data_as(vp))
    lib = L.lib()
    total = lib.hn_host_pack_panels(*args, None)
    packed = np.full(total, np.nan)
    assert lib.hn_host_pack_panels(*args, packed.ctypes.data_as(vp)) == total
    assert not np.isnan(packed).any()
    dense = tri.toarray()
    checked = 0
    for t in range(plan["ntasks"]):
        if kind[t] not in (0, 2):
            assert off[t] == -1
            continue
        b0, bw, pw = int(r0[t]), int(w[t]), int(rw[t])
        pos = int(off[t])
        nrect = (pw + 31) // 32
        if pw:  # rectangle panels first: predecessor columns in its tile order, all rows
            p0 = b0 - pw if lower else b0 + bw
            got = np.zeros((bw, pw))
            for q in range(nrect):
                c0 = 32 * q if lower else 32 * (nrect - 1 - q)
                tw = min(32, pw - c0)
                rp = (bw + 1) & ~1
                panel = packed[pos:pos + 32 * rp].reshape(32, rp)
                got[:, c0:c0 + tw] = panel[:tw, :bw].T
                pos += 32 * rp
            np.testing.assert_array_equal(got, dense[b0:b0 + bw, p0:p0 + pw])
            assert (got != 0).all()  # dense coupling
        got = np.zeros((bw, bw))
        for tt in range((bw + 31) // 32):
            t0, tw, rbase, rows, rp = _panel_geom(lower, bw, tt)
            panel = packed[pos:pos + 32 * rp].reshape(32, rp)
            assert pos % 2 == 0 and not panel[tw:].any()  # 16-byte aligned, missing columns zero
            got[rbase:rbase + rows, t0:t0 + tw] = panel[:tw, :rows].T
            pos += 32 * rp
        want = np.tril(dense[b0:b0 + bw, b0:b0 + bw], -1) if lower else np.triu(dense[b0:b0 + bw, b0:b0 + bw], 1)
        np.testing.assert_array_equal(got, want)
        checked += bw > 32
    assert checked > 0


def test_run_builds_the_domain_spec_for_cold_origins(monkeypatch):
    """run(config, nodeset=...) builds the domain spec before cold_origins(spec) (reference
    solver.py:412-415), with the package's own build_domain: obstacle cases read
    spec.obstacles there."""
    import paper_2303_01760_b200 as hn
    from paper_2303_01760_b200 import solver as S

    class Reached(Exception):
        pass

    seen = {}

    class Cfg(hn.CaseConfig):
        def cold_origins(self, spec):
            seen["spec"] = spec
            seen["cold"] = super().cold_origins(spec)
            raise Reached

    with pytest.raises(Reached):
        S.run(Cfg(case="dvd", h_r=0.05), nodeset=nodesets.jittered_box(8, seed=0))
    assert isinstance(seen["spec"], hn.DomainSpec) and seen["cold"] == {"wall:x-"}
    # (the obstacle case, whose placement runs on the device, is covered by
    # tests/test_gpu_solver.py::test_run_obstacle_case_with_precomputed_node_set)


def test_write_outputs_matches_reference_artifacts(tmp_path):
    """solver.write_outputs writes the reference bench layer's files and columns
    (pkg/src/hybridnodes/bench.py:28-44) from a RunResult (no GPU needed)."""
    import csv

    from paper_2303_01760_b200 import nodesets
    from paper_2303_01760_b200.operators import FieldState
    from paper_2303_01760_b200.solver import RunResult, write_outputs
    ns = nodesets.jittered_box(8, seed=1)
    n = len(ns)
    st = FieldState(np.ones((n, 2)), np.arange(n, dtype=float), np.full(n, 0.5))
    res = RunResult(case="dvd", discretization="hybrid", final_nu=1.2, nu_steps=np.array([10, 20]),
                    nu_times=np.array([0.1, 0.2]), nu_values=np.array([1.1, 1.2]), counts=(0, n, 0), n_total=n,
                    timings={"stepping": 2.0, "nodegen": 0.5}, dt=0.01, steps=20, t_final=0.25, state=st,
                    nodeset=ns)
    write_outputs(res, tmp_path / "out")
    rows = list(csv.reader(open(tmp_path / "out" / "nu_series.csv")))
    assert rows[0] == ["step", "t", "Nu"] and rows[2] == ["20", "0.2", "1.2"]
    rows = list(csv.reader(open(tmp_path / "out" / "timings.csv")))
    assert rows == [["phase", "seconds"], ["nodegen", "0.5"], ["stepping", "2.0"]]
    rows = list(csv.reader(open(tmp_path / "out" / "fields_0p25.csv")))
    assert rows[0] == ["x", "y", "u", "v", "p", "T", "h"] and len(rows) == n + 1
    np.testing.assert_allclose(np.array(rows[1:], dtype=float)[:, :2], ns.positions)


@pytest.mark.parametrize("keep", [3, 8, 20])
def test_dense_groups_host_arrays_solve_both_factors(keep):
    """The dense-group setup (solver.dense_group_runs / plan_groups / group_arrays, pure numpy)
    emulated in numpy exactly as csrc/pressure.cu executes it: the task rows by substitution
    (chosen rows empty), then per phase the coupling product and the row-packed inverse
    triangles -- against scipy's triangular solves, for L (groups last) and U (groups first)."""
    from scipy.sparse import linalg as spla

    from paper_2303_01760_b200.solver import (dense_group_runs, group_arrays, group_task_matrix, plan_groups,
                                              plan_supernodal_blocks)
    n = 700
    a = sp.random(n, n, density=0.012, random_state=3, format="csc") + sp.eye(n) * 3
    lu = spla.splu(a.tocsc())
    Ls = sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr")
    Us = sp.triu(sp.csr_matrix(lu.U), k=1, format="csr")
    Ls.sort_indices()
    Us.sort_indices()
    udiag = sp.csr_matrix(lu.U).diagonal()
    full = plan_supernodal_blocks(Ls, True)
    assert full["depth"] > keep + 4
    groups = dense_group_runs(Ls, full, keep, upper=Us)
    assert groups is not None
    rng = np.random.default_rng(0)
    for m, lower in ((Ls, True), (Us, False)):
        g = plan_groups(m, groups, lower)
        arr = group_arrays(m, g, lower)
        chosen = g["chosen"]
        # closure: no other row of L reads a chosen row; a chosen row of U reads only chosen rows
        rows_of = np.repeat(np.arange(n), np.diff(m.indptr))
        if lower:
            assert not chosen[m.indices[~chosen[rows_of]]].any()
        else:
            assert chosen[m.indices[chosen[rows_of]]].all()
        full_tri = (m + sp.eye(n)) if lower else (m + sp.diags(udiag))
        b = rng.normal(size=n)
        want = spsolve_triangular(full_tri.tocsr(), b, lower=lower)
        # inverse triangles, row-packed in execution order
        inv = np.zeros(arr["inv_entries"])
        for k in g["order"]:
            s0, s1 = int(g["starts"][k]), int(g["ends"][k])
            blk = full_tri.tocsr()[s0:s1, s0:s1].toarray()
            x = np.linalg.inv(blk)
            mask = np.tril(np.ones_like(x, dtype=bool)) if lower else np.triu(np.ones_like(x, dtype=bool))
            o = int(arr["run_off"][k])
            inv[o: o + mask.sum()] = x[mask]
        x = np.full(n, np.nan)
        rhs = b.copy()

        def phases():
            y = np.full(n, np.nan)
            for ph in range(len(g["phase_ptr"]) - 1):
                q0, q1 = int(g["phase_ptr"][ph]), int(g["phase_ptr"][ph + 1])
                for q in range(q0, q1):  # group_coupling_kernel
                    e0, e1 = arr["cpl_ptr"][q], arr["cpl_ptr"][q + 1]
                    xv = x[arr["cpl_cols"][e0:e1]]
                    assert not np.isnan(xv).any(), "coupling read an unsolved row"
                    y[g["rows"][q]] = rhs[g["rows"][q]] - np.dot(arr["cpl_vals"][e0:e1], xv)
                for q in range(q0, q1):  # group_gemv_kernel
                    o, c, ys = int(arr["g_off"][q]), int(arr["g_cnt"][q]), int(arr["g_ystart"][q])
                    x[g["rows"][q]] = np.dot(inv[o: o + c], y[ys: ys + c])
                    if not lower:
                        rhs[g["rows"][q]] = x[g["rows"][q]]  # echo

        lead = group_task_matrix(m, chosen)
        assert not np.diff(lead.indptr)[chosen].any()            # chosen rows are empty

        def tasks():  # the task kernel's rows (x = rhs / 1 on the empty chosen rows)
            order = range(n) if lower else range(n - 1, -1, -1)
            for i in order:
                c = lead.indices[lead.indptr[i]: lead.indptr[i + 1]]
                v = lead.data[lead.indptr[i]: lead.indptr[i + 1]]
                assert not np.isnan(x[c]).any()
                x[i] = (rhs[i] - np.dot(v, x[c])) / (1.0 if lower or chosen[i] else udiag[i])

        if lower:
            tasks()
            phases()
        else:
            phases()
            tasks()
        np.testing.assert_allclose(x, want, rtol=1e-8, atol=1e-10)
