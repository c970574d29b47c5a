"""Time the kNN query on the default grid vs the fine (query-spacing) grid (dev tool)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402
from paper_2303_01760_b200._device import DeviceNodes  # noqa: E402


def main():
    t = L.torch()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    flush = L.empty(32 << 20, t.float64)
    for name, ns, n in (("config1", nodesets.jittered_box(315, seed=1), 12),
                        ("config2", nodesets.hybrid_hole_2d(500, seed=2), 12),
                        ("config4", nodesets.hybrid_sphere_3d(94, seed=4, refine=2.8), 20)):
        dn = DeviceNodes(ns)
        rows = L.to_device(np.nonzero(ns.kind == 1)[0].astype(np.int32))
        res = {}
        for fine in (False, True):
            out = dn.knn(n, rows=rows, fine=fine)
            ts = []
            for _ in range(5):
                flush.fill_(1.0)
                e0.record(); out = dn.knn(n, rows=rows, fine=fine); e1.record(); t.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[fine] = out.cpu().numpy()
            print(f"{name} fine={fine} (cell {dn.fine_cell if fine else dn.cell}): {np.median(ts) * 1e3:.1f} us "
                  f"for {rows.numel()} queries n={n}", flush=True)
        print(f"{name} identical: {np.array_equal(res[False], res[True])}", flush=True)


if __name__ == "__main__":
    main()
