"""Generate golden vectors by running the REFERENCE itself (test infrastructure).

Usage (in the build container, where /root/reference exists):
    OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/make_golden.py

Imports the reference package from /root/reference/pkg/src (read-only, never copied)
and writes tests/golden/<case>.npz: the input node set and the reference's outputs
(method, stencil indices, weights, applied fields, boundary/Nusselt tables, Poisson
matrix, fields after k explicit steps).  The GPU box has no /root/reference: tests use
these committed fixtures and the oracle port (oracle/hn_oracle.py).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
OUT = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(REF))

from hybridnodes import approx as R_approx  # noqa: E402
from hybridnodes import nodegen as R_nodegen  # noqa: E402
from hybridnodes import operators as R_ops  # noqa: E402
from hybridnodes import solver as R_solver  # noqa: E402
from hybridnodes.config import CaseConfig, build_domain  # noqa: E402

from paper_2303_01760_b200 import nodesets  # noqa: E402
from paper_2303_01760_b200.nodegen import NodeSet as HNodeSet  # noqa: E402


def ref_nodeset(ns) -> "R_nodegen.NodeSet":
    """The same node set as a reference NodeSet object."""
    lat = None
    if ns.lattice is not None:
        lat = R_nodegen.LatticeInfo(np.asarray(ns.lattice.origin), np.asarray(ns.lattice.step),
                                    tuple(ns.lattice.cells), np.asarray(ns.lattice.grid).copy())
    return R_nodegen.NodeSet(ns.positions, ns.spacing, ns.kind, ns.role, ns.bc_value, ns.normals, list(ns.origin),
                             lat, None if ns.lattice_idx is None else np.asarray(ns.lattice_idx).copy())


def ours(ns) -> HNodeSet:
    lat = None
    from paper_2303_01760_b200.nodegen import LatticeInfo
    if ns.lattice is not None:
        lat = LatticeInfo(np.asarray(ns.lattice.origin), np.asarray(ns.lattice.step), tuple(ns.lattice.cells),
                          np.asarray(ns.lattice.grid).copy())
    return HNodeSet(ns.positions, ns.spacing, ns.kind, ns.role, ns.bc_value, ns.normals, list(ns.origin), lat,
                    None if ns.lattice_idx is None else np.asarray(ns.lattice_idx).copy())


def field(pos, seed=7):
    return nodesets.sinusoid_field(pos, seed=seed)


def weights_block(rns, dim, prefix, ops_names, rbf_n=None):
    ops = [R_approx.Laplacian()] + [R_approx.Partial(a) for a in range(dim)]
    saved = dict(R_approx.RBF_SIZE)
    if rbf_n is not None:
        R_approx.RBF_SIZE[dim] = rbf_n
    try:
        table = R_approx.compute_weights(rns, ops)
    finally:
        R_approx.RBF_SIZE.clear()
        R_approx.RBF_SIZE.update(saved)
    out = {f"{prefix}method": table.method, f"{prefix}indices": table.indices, f"{prefix}sizes": table.sizes}
    f = field(rns.positions)
    out[f"{prefix}field"] = f
    for name, op in zip(ops_names, ops):
        out[f"{prefix}w_{name}"] = table.weights[op]
        out[f"{prefix}apply_{name}"] = R_ops.assemble(rns, table, op).apply(f)
    return out, table


def boundary_block(rns, prefix, cold_origins, size_override=None):
    dim = rns.dim
    saved = dict(R_approx.RBF_SIZE)
    if size_override is not None:
        R_approx.RBF_SIZE[dim] = size_override
    try:
        bidx = np.nonzero(rns.boundary_mask)[0]
        bg = R_approx.boundary_partial_table(rns, bidx, exclude=rns.boundary_mask)
        cold = np.array([i for i in bidx if rns.origin[i] in cold_origins], dtype=np.int64)
        nt = R_approx.normal_derivative_table(rns, cold) if len(cold) else None
    finally:
        R_approx.RBF_SIZE.clear()
        R_approx.RBF_SIZE.update(saved)
    out = {f"{prefix}bgrad_indices": bg.indices, f"{prefix}bgrad_sizes": bg.sizes}
    for a in range(dim):
        out[f"{prefix}bgrad_w_d{a}"] = bg.weights[R_approx.Partial(a)]
    if nt is not None:
        out[f"{prefix}nu_rows"] = cold
        out[f"{prefix}nu_indices"] = nt.indices
        out[f"{prefix}nu_w"] = nt.weights["normal"]
    return out


def steps_block(rns, prefix, n_steps, Ra, Pr, seed=11, table_rbf_n=None, dissipation=0.0):
    """Replicates run()'s loop body (solver.py:439-452) from T = (x - 0.5) + 1e-3 noise."""
    dim = rns.dim
    settings = R_solver.PoissonSolveSettings()
    saved = dict(R_approx.RBF_SIZE)
    try:
        if table_rbf_n is not None:
            # interior n from table_rbf_n, boundary tables at the reference default (H9)
            orig = R_approx.compute_weights

            def cw(ns, ops, with_kappa=False, tree=None):
                R_approx.RBF_SIZE[dim] = table_rbf_n
                try:
                    return orig(ns, ops, with_kappa, tree)
                finally:
                    R_approx.RBF_SIZE[dim] = saved[dim]

            R_solver.compute_weights = cw
        ops = R_solver.build_operators(rns, {"wall:x-"}, settings)
    finally:
        R_solver.compute_weights = R_approx.compute_weights
        R_approx.RBF_SIZE.clear()
        R_approx.RBF_SIZE.update(saved)
    params = R_solver.PhysicsParams(Ra, Pr, t_ref=0.0, dissipation=dissipation)
    dt = R_solver.TimeControls.from_spacing(float(np.min(rns.spacing)), 1.0, Ra=Ra).dt
    rng = np.random.default_rng(seed)
    n = len(rns)
    state = R_ops.FieldState.zeros(n, dim)
    state.temperature[:] = (rns.positions[:, 0] - 0.5) + 1e-3 * rng.normal(size=n)
    R_solver.apply_temperature_bc(state.temperature, ops)
    out = {f"{prefix}T0": state.temperature.copy(), f"{prefix}dt": dt, f"{prefix}Ra": Ra, f"{prefix}Pr": Pr,
           f"{prefix}gauge": ops.gauge, f"{prefix}poisson_indptr": ops.poisson_matrix.indptr,
           f"{prefix}poisson_indices": ops.poisson_matrix.indices, f"{prefix}poisson_data": ops.poisson_matrix.data}
    p_prev = None
    for k in range(1, n_steps + 1):
        vstar = R_solver.momentum_predict(state, ops, params, dt)
        if k == 1:
            out[f"{prefix}vstar1_raw"] = vstar.copy()
        R_solver.apply_velocity_bc(vstar, ops)
        p = R_solver.pressure_solve(vstar, ops, settings, dt, x0=p_prev)
        v_new = R_solver.velocity_correct(vstar, p, ops, dt)
        state.velocity = v_new
        state.pressure = p
        p_prev = p
        state.temperature = R_solver.temperature_step(state, ops, dt, params.dissipation)
        if k == 1:
            out[f"{prefix}v1"], out[f"{prefix}T1"], out[f"{prefix}p1"] = v_new.copy(), state.temperature.copy(), p.copy()
    out[f"{prefix}vK"], out[f"{prefix}TK"], out[f"{prefix}pK"] = (state.velocity.copy(), state.temperature.copy(),
                                                                 state.pressure.copy())
    out[f"{prefix}steps"] = n_steps
    out[f"{prefix}dissipation"] = dissipation
    out[f"{prefix}nuK"] = R_solver.nusselt_average(state, ops)
    return out


def save(name, ns, blocks):
    arrs = {}
    for k, v in ours(ns).to_arrays().items():
        arrs[f"ns_{k}"] = v
    for b in blocks:
        arrs.update(b)
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **arrs)
    print(f"{name}: N={len(ns)} -> {OUT / (name + '.npz')} ({(OUT / (name + '.npz')).stat().st_size / 1e3:.0f} kB)")


def main():
    names2 = ["lap", "d0", "d1"]
    names3 = ["lap", "d0", "d1", "d2"]

    # 1) the reference's own operator-test fixture (tests/conftest.py:15-20): hybrid dvd
    cfg = CaseConfig(case="dvd", h_r=0.0398)
    ns = R_nodegen.hybrid_discretize(cfg, build_domain(cfg))
    w, _ = weights_block(ns, 2, "", names2)
    save("dvd_coarse", ns, [w, boundary_block(ns, "", {"wall:x-"}), steps_block(ns, "", 20, 1e6, 0.71),
                            steps_block(ns, "hd_", 20, 1e6, 0.71, dissipation=0.05)])

    # 2) the reference's pure-scattered fixture (conftest.py:31-36)
    cfg = CaseConfig(case="dvd", h_r=0.05, discretization="pure-scattered")
    ns = R_nodegen.hybrid_discretize(cfg, build_domain(cfg))
    w, _ = weights_block(ns, 2, "", names2)
    save("scattered_cloud", ns, [w])

    # 3) config 0 generator: the reference's dvd pure-regular set, small (h = 1/49) and our twin
    cfg = CaseConfig(case="dvd", discretization="pure-regular", h_r=1 / 49)
    ns = R_nodegen.hybrid_discretize(cfg, build_domain(cfg))
    w, _ = weights_block(ns, 2, "", names2)
    save("config0_small_ref", ns, [w])

    # 4) builder generators at reduced size, reference computes everything
    for name, gen in (("config0_small", lambda: nodesets.regular_box(49)),
                      ("config1_small", lambda: nodesets.jittered_box(40, seed=1)),
                      ("config2_small", lambda: nodesets.hybrid_hole_2d(60, seed=2))):
        hns = gen()
        rns = ref_nodeset(hns)
        w, _ = weights_block(rns, 2, "", names2)
        blocks = [w, boundary_block(rns, "", {"wall:x-"})]
        if name == "config2_small":
            blocks.append(steps_block(rns, "", 10, 1e6, 0.71))
        save(name, hns, blocks)

    # 5) 3D, reduced size: interior n = 20 (BASELINE) with boundary tables at n = 30 (H9)
    hns = nodesets.hybrid_sphere_3d(12, seed=4, refine=2.8)
    rns = ref_nodeset(hns)
    w20, _ = weights_block(rns, 3, "", names3, rbf_n=20)
    w30, _ = weights_block(rns, 3, "n30_", names3, rbf_n=30)
    save("config4_small", hns, [w20, w30, boundary_block(rns, "", {"wall:x-"}),
                                steps_block(rns, "", 3, 1e5, 0.71, table_rbf_n=20)])


if __name__ == "__main__":
    main()
