"""Repeat the device LU preconditioner solve many times on config-3 factors and check every
result against the first one (bitwise) and against host SuperLU (dev tool: race hunting)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402


def main():
    t = L.torch()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 400
    ns = nodesets.hybrid_hole_2d(M, seed=2)
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings())
    dlu = ops._d_lu
    n = dlu.n
    rng = np.random.default_rng(0)
    bh = rng.normal(size=n)
    xref = ops.poisson_precond.matvec(bh)
    b = L.to_device(bh)
    x = L.empty(n, t.float64)
    first = None
    bad = 0
    worst = 0.0
    for i in range(reps):
        x.fill_(np.nan)
        dlu.solve(b, x)
        xh = x.cpu().numpy()
        if first is None:
            first = xh.copy()
        err = float(np.max(np.abs(xh - xref)) / np.max(np.abs(xref)))
        worst = max(worst, err)
        if not np.array_equal(xh, first):
            bad += 1
            d = np.nonzero(xh != first)[0]
            if bad <= 5:
                print(f"rep {i}: {len(d)} entries differ from rep 0 (first {d[:8]}), rel err vs host {err:.3e}",
                      flush=True)
    print(f"n={n}: {bad}/{reps} reps differ from rep 0; worst rel err vs host SuperLU {worst:.3e}", flush=True)

    # the same in the stepping context: matvec counts per step
    dt = hn.TimeControls.from_spacing(float(np.min(ns.spacing)), 1.0, Ra=1e6).dt
    T0 = (ns.positions[:, 0] - 0.5) + 1e-3 * np.random.default_rng(3).normal(size=len(ns))
    st = hn.FieldState(np.zeros((len(ns), 2)), np.zeros(len(ns)), T0)
    hn.apply_temperature_bc(st.temperature, ops)
    stepper = hn.DeviceStepper(ops, hn.PhysicsParams(1e6, 0.71), hn.PoissonSolveSettings(), dt, st)
    its = []
    for k in range(int(sys.argv[3]) if len(sys.argv) > 3 else 80):
        m0 = stepper.solver.matvecs
        try:
            stepper.step()
        except Exception as e:  # noqa: BLE001
            print(f"step {k}: {type(e).__name__}: {e}", flush=True)
            break
        its.append(stepper.solver.matvecs - m0)
    print("matvecs per step:", its, flush=True)


if __name__ == "__main__":
    main()
