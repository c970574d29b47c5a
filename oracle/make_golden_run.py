"""Golden vectors for the run() loop, made by running the REFERENCE's own solver.run
(test infrastructure; /root/reference must exist, i.e. this container).

    OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/make_golden_run.py

Writes tests/golden/run_jittered.npz:
  * a normal run (reference solver.py:395-490) of the dvd case on a tie-free jittered node set
    (no exact-tie boundary rows, so the GPU's own stencils are the
    reference's): Nu series, step count, final fields, divergence samples;
  * a diverging run of the same set (Pr = 60: the explicit viscous term is unstable at the
    reference's dt) and the step and node of the reference's SolverDivergenceError.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from hybridnodes import solver as R_solver  # noqa: E402
from hybridnodes.config import CaseConfig  # noqa: E402
from hybridnodes.errors import SolverDivergenceError  # noqa: E402

from oracle.make_golden import ref_nodeset  # noqa: E402
from paper_2303_01760_b200 import nodesets  # noqa: E402

RUN = dict(case="dvd", discretization="hybrid", Ra=1e6, Pr=0.71, t_cold=-0.5, t_hot=0.5, t_init=0.0,
           t_end=2.4e-3, nu_stride=20)
DIVERGE = dict(RUN, Pr=60.0, t_end=0.04)


def main():
    ns = nodesets.jittered_box(30, seed=1)
    out = {f"ns_{k}": v for k, v in ns.to_arrays().items()}
    res = R_solver.run(CaseConfig(**RUN), nodeset=ref_nodeset(ns))
    out.update(run_cfg=np.array([RUN["Ra"], RUN["Pr"], RUN["t_cold"], RUN["t_hot"], RUN["t_init"], RUN["t_end"],
                                 RUN["nu_stride"]]),
               run_steps=res.steps, run_dt=res.dt, run_nu_steps=res.nu_steps, run_nu_values=res.nu_values,
               run_v=res.state.velocity, run_T=res.state.temperature, run_p=res.state.pressure,
               run_div=np.asarray(res.diagnostics["divergence_samples"], dtype=float))
    try:
        R_solver.run(CaseConfig(**DIVERGE), nodeset=ref_nodeset(ns))
        raise SystemExit("the diverging configuration did not diverge")
    except SolverDivergenceError as e:
        out.update(div_cfg=np.array([DIVERGE["Pr"], DIVERGE["t_end"]]), div_step=e.step, div_node=e.node)
        print("reference diverged at step", e.step, "node", e.node)
    path = ROOT / "tests" / "golden" / "run_jittered.npz"
    np.savez_compressed(path, **out)
    print("wrote", path, "steps", res.steps, "Nu", res.final_nu)


if __name__ == "__main__":
    main()
