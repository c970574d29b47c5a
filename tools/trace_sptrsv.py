"""Record the per-task timeline of the supernodal L and U solves on config 3 (dev tool);
writes gpurun_out/trace_sptrsv.npz for offline analysis."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
# the trace hook only exists in the dev build (python -m paper_2303_01760_b200._build --trace)
os.environ.setdefault("HN_LIB_PATH", str(ROOT / "paper_2303_01760_b200" / "libhn_trace.so"))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402


def main():
    t = L.torch()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    ns = nodesets.hybrid_hole_2d(M, seed=2)
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings())
    lu = ops._d_lu
    n1 = lu.n
    b = L.to_device(np.random.default_rng(0).normal(size=n1))
    y = L.empty(n1, t.float64)
    out = {}
    s = L.stream_handle()
    for name, sch, m, dg in (("L", lu.sL, lu.L, None), ("U", lu.sU, lu.U, lu.diag)):
        tr = L.zeros(4 * sch.kind.numel(), t.int64)
        lu._tri(sch, m, dg, b, y, s)  # warm
        t.cuda.synchronize()
        L.lib().hn_debug_sptrsv_trace(L.ptr(tr))
        e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        e0.record()
        lu._tri(sch, m, dg, b, y, s)
        e1.record()
        t.cuda.synchronize()
        L.lib().hn_debug_sptrsv_trace(None)
        out[name + "_trace"] = tr.cpu().numpy().reshape(-1, 4)[: sch.ntasks]
        for k in ("kind", "r0", "w", "rb", "rc"):
            out[name + "_" + k] = getattr(sch, k).cpu().numpy()
        out[name + "_ms"] = e0.elapsed_time(e1)
        print(name, "solve ms", out[name + "_ms"], "tasks", sch.ntasks, flush=True)
    out["rowptr_L"] = lu.L.rowptr.cpu().numpy()
    out["rowptr_U"] = lu.U.rowptr.cpu().numpy()
    np.savez_compressed(Path(__file__).resolve().parents[1] / "gpurun_out" / "trace_sptrsv.npz", **out)


if __name__ == "__main__":
    main()
