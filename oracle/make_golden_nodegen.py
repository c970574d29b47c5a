"""Golden node sets for the device generator, made by running the
REFERENCE's own generator (test infrastructure; run in the build container):

    OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/make_golden_nodegen.py

Imports hybridnodes from /root/reference/pkg/src (read-only, never copied) and writes
tests/golden/nodegen_<case>.npz: the NodeSet arrays of hybrid_discretize(config) plus the
obstacle layout build_domain(config) chose (kind, parameters, temperature), and the
reference's regular_fill / carve_transition / scattered_fill outputs for the API cases of
its own tests (tests/test_nodegen.py).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
sys.path.insert(0, "/root/reference/pkg/src")

from hybridnodes import nodegen as R  # noqa: E402
from hybridnodes.config import CaseConfig, build_domain  # noqa: E402
from hybridnodes.geometry import Circle, DomainSpec, Obstacle  # noqa: E402

# name -> CaseConfig overrides (sizes kept small: the fixtures are committed)
CASES = {
    "dvd_h0398": dict(case="dvd", h_r=0.0398),
    "dvd_h01": dict(case="dvd", h_r=0.01),
    "dvd_pure_scattered": dict(case="dvd", h_r=0.05, discretization="pure-scattered"),
    "dvd_pure_regular": dict(case="dvd", h_r=0.05, discretization="pure-regular"),
    "split_vertical": dict(case="dvd-split", h_r=0.02, delta_h=8, split_orientation="vertical"),
    "split_full": dict(case="dvd-split", h_r=0.05, delta_h=1 / 0.05),
    "custom_box": dict(case="custom", h_r=0.1),
    "spheres3d_h05": dict(case="spheres3d", h_r=0.05),
    "spheres3d_two_seed5": dict(case="spheres3d", h_r=0.04, rng_seed=5, n_spheres=2, sphere_radius_max=0.12),
    "obstacles2d_h02": dict(case="obstacles2d", h_r=0.02),
}


def layout(spec):
    kinds, par, temp = [], np.zeros((len(spec.obstacles), 8)), []
    for j, obs in enumerate(spec.obstacles):
        sh = obs.shape
        if hasattr(sh, "lobes"):
            kinds.append(1)
            par[j, :6] = (*sh.center, sh.mean_radius, sh.amplitude, sh.lobes, sh.phase)
        else:
            kinds.append(0)
            par[j, :len(sh.center)] = sh.center
            par[j, len(sh.center)] = sh.radius
        temp.append(np.nan if obs.temperature is None else obs.temperature)
    return np.asarray(kinds, np.int64), par, np.asarray(temp, float)


def save_nodeset(path, ns, **extra):
    np.savez_compressed(path, positions=ns.positions, spacing=ns.spacing, kind=ns.kind, role=ns.role,
                        bc_value=ns.bc_value, normals=ns.normals, origin=np.array(ns.origin, dtype="U16"),
                        lattice_origin=ns.lattice.origin, lattice_step=ns.lattice.step,
                        lattice_cells=np.asarray(ns.lattice.cells, np.int64), lattice_grid=ns.lattice.grid,
                        lattice_idx=ns.lattice_idx, **extra)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    for name, kw in CASES.items():
        cfg = CaseConfig(**kw)
        spec = build_domain(cfg)
        ns = R.hybrid_discretize(cfg, spec)
        k, p, t = layout(spec)
        save_nodeset(OUT / f"nodegen_{name}.npz", ns, obs_kind=k, obs_par=p, obs_temp=t,
                     config=np.array(repr(sorted(kw.items()))))
        print(name, len(ns), ns.counts, flush=True)
    # API cases of the reference's own tests (tests/test_nodegen.py:18-100)
    box = DomainSpec(np.zeros(2), np.ones(2))
    circ = DomainSpec(np.zeros(2), np.ones(2), (Obstacle(Circle((0.5, 0.5), 0.2), 0.0),))
    seeds = np.array([[0.5, 0.0], [0.0, 0.5], [1.0, 0.5], [0.5, 1.0]])
    sf = R.SpacingFunction(0.1, 0.1, 0.0)
    graded = R.SpacingFunction(0.03, 0.01, 4.0, circ.obstacle_distance)
    fill = R.regular_fill(circ, 0.05)
    carved = R.carve_transition(fill, circ, 2.0, 0.05)
    probe = np.random.default_rng(3).uniform(0, 1, size=(4000, 2))
    np.savez_compressed(
        OUT / "nodegen_api.npz",
        fill_pos=fill.positions, fill_idx=fill.indices, fill_step=fill.step,
        carved_pos=carved.positions,
        sf11=R.scattered_fill(box, seeds, sf, rng_seed=11), sf12=R.scattered_fill(box, seeds, sf, rng_seed=12),
        sf_graded=R.scattered_fill(circ, seeds, graded, rng_seed=4),
        probe=probe, probe_sd=circ.signed_distance(probe), probe_obs=circ.obstacle_distance(probe),
        probe_box=circ.box_signed_distance(probe), probe_h=graded(probe))
    print("api ok")


if __name__ == "__main__":
    main()
