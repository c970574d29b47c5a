"""Time the L and U supernodal solves and one full preconditioner application on config 3 for a
list of dense-group depths (block levels left to the task chain; 0 = no groups), with the distance to SuperLU's own solve (dev tool; CUDA events,
median of 20).
  python tools/time_trisolve.py [M=500] [keep_levels, e.g. 0,60,40,30] [inverse modes, e.g. 0,1,2] [helper_nnz, e.g. 4096,16384]"""
import sys
import time
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
    ts = []
    for _ in range(reps):
        e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    t = L.torch()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    tails = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 60, 50, 40, 30]
    modes = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [None]
    helpers = [int(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else [4096]
    extra = [dict(kv.split("=") for kv in a.split(";")) for a in sys.argv[5:]] or [{}]  # plan kwargs, e.g. cap=128;batch=4
    extra = [{k: int(v) for k, v in e.items()} for e in extra]
    ns = nodesets.hybrid_hole_2d(M, seed=2)
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings(), factorize=True)
    host_lu = spla.splu(ops.poisson_matrix.tocsc())
    rhs = np.random.default_rng(0).normal(size=host_lu.shape[0])
    ref = host_lu.solve(rhs)
    b = L.to_device(rhs)
    for tail, mode, hz, kw in [(a, b, c, e) for a in tails for b in modes for c in helpers for e in extra]:
        t0 = time.perf_counter()
        lu = _DeviceLU(host_lu, keep_levels=tail, inverse=mode, helper_nnz=hz, **kw)
        t.cuda.synchronize()
        setup = time.perf_counter() - t0
        x = L.empty(lu.n, t.float64)
        s = L.stream_handle()
        tl = timeit(lambda: lu._tri(lu.sL, lu.L, None, b, lu.z, s))
        bu = b.clone()  # an upper plan with dense groups overwrites the groups' rhs entries
        tu = timeit(lambda: lu._tri(lu.sU, lu.U, lu.diag, bu, lu.w, s))
        tp = timeit(lambda: lu.solve(b, x))
        err = np.abs(x.cpu().numpy() - ref).max() / np.abs(ref).max()
        print(f"keep {tail:3d} rows {lu.group_rows:6d} phases {lu.sL.n_phases}/{lu.sU.n_phases} inverse {lu.sL.inverse} helper {hz} {kw} tasks {lu.sL.ntasks}/{lu.sU.ntasks}: L {tl:.3f} ms  U {tu:.3f} ms  precond {tp:.3f} ms  vs SuperLU {err:.2e}  "
              f"depth L {lu.sL.depth} U {lu.sU.depth}  bytes {lu.solve_bytes / 1e6:.0f} MB  setup {setup:.1f} s",
              flush=True)
        del lu, x
        t.cuda.empty_cache()


if __name__ == "__main__":
    main()
