"""Time kNN query variants (ring traversal vs box pass at several radii, default vs fine
grid) on the scattered queries of configs 1, 2 and 4, checking identical results (dev tool)."""
import ctypes as C
import os
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
if "--trace" in sys.argv:  # dev build with the warp-kNN fallback counters
    os.environ.setdefault("HN_LIB_PATH", str(ROOT / "paper_2303_01760_b200" / "libhn_trace.so"))
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402
from paper_2303_01760_b200._device import DeviceNodes  # noqa: E402


def main():
    t = L.torch()
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    variants = [int(v) for v in (args[0] if args else "1,0,2,3").split(",")]
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    flush = L.empty(32 << 20, t.float64)
    cases = [("config4", nodesets.hybrid_sphere_3d(94, seed=4, refine=2.8), 20)]
    if "--c4" in sys.argv:  # 3D only, also the reference-default n = 30
        cases.append(("config4", cases[0][1], 30))
    else:
        cases = [("config1", nodesets.jittered_box(315, seed=1), 12),
                 ("config2", nodesets.hybrid_hole_2d(500, seed=2), 12)] + cases
    for name, ns, n in cases:
        dn = DeviceNodes(ns)
        rows = L.to_device(np.nonzero(ns.kind == 1)[0].astype(np.int32))
        ref = None
        for v in variants:
            L.lib().hn_knn_set_variant(v)
            for fine in (False, True):
                out = dn.knn(n, rows=rows, fine=fine)
                ts = []
                for _ in range(5):
                    flush.fill_(1.0)
                    e0.record(); out = dn.knn(n, rows=rows, fine=fine); e1.record(); t.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                o = out.cpu().numpy()
                if ref is None:
                    ref = o
                fbs = ""
                if "--trace" in sys.argv:
                    st = (C.c_ulonglong * 4)()
                    L.lib().hn_debug_knn_fallbacks(st)
                    fbs = f"  fallbacks/call {st[0] // 6} (>32: {st[1] // 6}, <n: {st[2] // 6}, nth>r: {st[3] // 6})"
                print(f"{name} variant {v} fine={fine}: {np.median(ts) * 1e3:.1f} us for {rows.numel()} queries "
                      f"n={n}  identical={np.array_equal(o, ref)}{fbs}", flush=True)
        L.lib().hn_knn_set_variant(0)


if __name__ == "__main__":
    main()
