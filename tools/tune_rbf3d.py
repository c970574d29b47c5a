"""Time the 3D RBF weight kernel (n = 20 and 30, 4 ops) on config 4's scattered rows (dev tool)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01760_b200 import _lib as L  # noqa: E402
from paper_2303_01760_b200 import nodesets  # noqa: E402
from paper_2303_01760_b200._device import device_nodes  # noqa: E402


def main():
    t = L.torch()
    ns = nodesets.hybrid_sphere_3d(94, seed=4, refine=2.8)
    dn = device_nodes(ns)
    rows = np.nonzero(ns.kind == 1)[0]
    K = len(rows)
    kinds, axes, nrm = L.host_ints([0, 1, 1, 1]), L.host_ints([0, 0, 1, 2]), L.host_dbls([0] * 12)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    flush = L.empty(64 * 2 ** 20, t.float64)
    flops = {20: 24625, 30: 66000}
    for n in (20, 30):
        cache = Path(__file__).resolve().parents[1] / "gpurun_out" / f"st3d_{n}.npy"
        if cache.exists():  # A/B runs against an older libhn (HN_LIB_PATH) reuse the stencils
            st = L.to_device(np.load(cache))
        else:
            st = dn.knn(n, rows=L.to_device(rows.astype(np.int32)), fine=True)
            np.save(cache, st.cpu().numpy())
        oi = L.empty((n, K), t.int32)
        ow = L.empty((4, n, K), t.float64)
        info = L.zeros(K, t.int32)
        times = []
        for rep in range(6):
            flush.fill_(rep)
            e0.record()
            L.call("hn_weights_rbf", L.ptr(dn.pos), 3, L.ptr(st), K, n, 4, kinds, axes, nrm, None, None,
                   L.ptr(oi), L.ptr(ow), L.ptr(info), L.stream_handle())
            e1.record()
            t.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times[1:]))
        bad = int((info != 0).sum().item())
        print(f"3D n={n}: {ms * 1e3:.1f} us for {K} stencils, {K * flops[n] / ms / 1e9:.2f} TFLOP/s (LAPACK count), "
              f"singular {bad}, w checksum {float(ow.double().abs().sum()):.6e}", flush=True)


if __name__ == "__main__":
    main()
