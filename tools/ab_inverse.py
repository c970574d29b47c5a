"""A/B of the packed-panel trisolve with and without diagonal-tile inverses on config 3
(dev tool): per-solve time, distance to SuperLU's solve, and the field drift after K steps
against the substitution-only run.  Usage: python tools/ab_inverse.py [M] [steps]"""
import sys
from pathlib import Path

import numpy as np
from scipy.sparse import linalg as spla

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402
from paper_2303_01760_b200.solver import _DeviceLU  # noqa: E402


def timeit(fn, reps=20):
    t = L.torch()
    fn()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    t.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    t = L.torch()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    ns = nodesets.hybrid_hole_2d(M, seed=2)
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings())
    lu = spla.splu(ops.poisson_matrix.tocsc())
    n = lu.shape[0]
    b = np.random.default_rng(0).normal(size=n)
    ref = lu.solve(b)
    bd, xd = L.to_device(b), L.empty(n, t.float64)
    Ra, Pr = 1e6, 0.71
    dt = hn.TimeControls.from_spacing(float(np.min(ns.spacing)), 1.0, Ra=Ra).dt
    T0 = (ns.positions[:, 0] - 0.5) + 1e-3 * np.random.default_rng(3).normal(size=len(ns))
    fields = {}
    for mode in ((False, False), (True, False), (False, True), (True, True)):
        _DeviceLU.TILE_INVERSE_L, _DeviceLU.TILE_INVERSE_U = mode
        dlu = _DeviceLU(lu)
        s = L.stream_handle()
        tl = timeit(lambda: dlu._tri(dlu.sL, dlu.L, None, bd, dlu.z, s))
        bu = bd.clone()  # the upper solve with dense groups overwrites the groups' rhs entries
        tu = timeit(lambda: dlu._tri(dlu.sU, dlu.U, dlu.diag, bu, dlu.w, s))
        dlu.solve(bd, xd)
        err = np.abs(xd.cpu().numpy() - ref).max() / np.abs(ref).max()
        res = np.linalg.norm(ops.poisson_matrix @ xd.cpu().numpy() - b) / np.linalg.norm(b)
        ops._d_lu = dlu
        st = hn.FieldState(np.zeros((len(ns), 2)), np.zeros(len(ns)), T0.copy())
        hn.apply_temperature_bc(st.temperature, ops)
        stepper = hn.DeviceStepper(ops, hn.PhysicsParams(Ra, Pr), hn.PoissonSolveSettings(), dt, st)
        for _ in range(steps):
            stepper.step()
        fields[mode] = stepper.state()
        f0 = fields[(False, False)]
        drift = {k: float(np.abs(getattr(fields[mode], k) - getattr(f0, k)).max() / np.abs(getattr(f0, k)).max())
                 for k in ("velocity", "temperature", "pressure")}
        print(f"inverse L={mode[0]!s:5} U={mode[1]!s:5}  L {tl:.3f} ms  U {tu:.3f} ms  |x-superlu|/|x| {err:.2e}  "
              f"relres {res:.2e}  drift after {steps} steps {drift}", flush=True)


if __name__ == "__main__":
    main()
