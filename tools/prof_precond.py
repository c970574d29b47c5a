"""Time the device LU preconditioner (supernodal sync-free solves) on config 3 for planner /
launch variants, checking every variant against SuperLU (dev tool)."""
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets, solver  # noqa: E402


def host_csr(d, n):
    return sp.csr_matrix((d.vals.cpu().numpy(), d.cols.cpu().numpy(), d.rowptr.cpu().numpy()), shape=(n, n))


def main():
    t = L.torch()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    ns = nodesets.hybrid_hole_2d(M, seed=2)
    t0 = time.perf_counter()
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings())
    print(f"N={len(ns)} build_operators {time.perf_counter() - t0:.1f}s", flush=True)
    lu = ops._d_lu
    n1 = lu.n
    Lh, Uh = host_csr(lu.L, n1), host_csr(lu.U, n1)
    bh = np.random.default_rng(0).normal(size=n1)
    want = ops.poisson_precond.matvec(bh)
    b = L.to_device(bh)
    x = L.empty(n1, t.float64)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    caps = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "4096,512,256,128,64").split(",")]
    hel = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "16384").split(",")]
    brn = [int(v) for v in (sys.argv[4] if len(sys.argv) > 4 else "96").split(",")]
    for cap in caps:
     for helper in hel:
      for brow in brn:
        batch = 8
        t0 = time.perf_counter()
        lu.sL = solver._SuperSchedule(Lh, lower=True, batch=batch, cap=cap, helper_nnz=helper, batch_row_nnz=brow)
        lu.sU = solver._SuperSchedule(Uh, lower=False, batch=batch, cap=cap, helper_nnz=helper, batch_row_nnz=brow)
        plan_s = time.perf_counter() - t0
        for cps in (2,):
            lu.CTAS_PER_SM = cps
            lu.solve(b, x)
            t.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0.record()
                lu.solve(b, x)
                e1.record()
                t.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            err = np.abs(x.cpu().numpy() - want).max() / np.abs(want).max()
            print(f"cap {cap} helper {helper} batch_row_nnz {brow} ctas/SM {cps}: precond {np.median(ts):.3f} ms (min {min(ts):.3f})  tasks L "
                  f"{lu.sL.ntasks} U {lu.sU.ntasks}  rel err vs SuperLU {err:.1e}  (plan {plan_s:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
