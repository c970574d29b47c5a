"""Time launch-shape variants of the 2D RBF weight kernel on config 1 (dev tool)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01760_b200 import _lib as L  # noqa: E402
from paper_2303_01760_b200 import nodesets  # noqa: E402
from paper_2303_01760_b200._device import device_nodes  # noqa: E402


def main():
    t = L.torch()
    ns = nodesets.jittered_box(315, seed=1)
    dn = device_nodes(ns)
    rows = np.nonzero(ns.kind != 2)[0]
    st = dn.knn(12, rows=L.to_device(rows.astype(np.int32)))
    K = len(rows)
    kinds, axes, nrm = L.host_ints([0, 1, 1]), L.host_ints([0, 0, 1]), L.host_dbls([0] * 6)
    ref = None
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    flush = L.empty(64 * 2 ** 20, t.float64)  # 512 MB > L2
    for v in [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else '0,1,2,3,4,5'.split(','))]:
        L.lib().hn_weights_rbf_set_variant(v)
        oi = L.empty((12, K), t.int32)
        ow = L.empty((3, 12, K), t.float64)
        info = L.zeros(K, t.int32)
        times = []
        for rep in range(6):
            flush.fill_(rep)
            e0.record()
            L.call("hn_weights_rbf", L.ptr(dn.pos), 2, L.ptr(st), K, 12, 3, kinds, axes, nrm, None, None,
                   L.ptr(oi), L.ptr(ow), L.ptr(info), L.stream_handle())
            e1.record()
            t.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        w = ow.cpu().numpy()
        if ref is None:
            ref = w
        err = np.abs(w - ref).max() / np.abs(ref).max()
        ms = float(np.median(times[1:]))
        print(f"variant {v}: {ms * 1e3:.1f} us  {K * 5613 / ms / 1e9:.2f} TFLOP/s  maxdiff vs v0 {err:.2e}", flush=True)
    L.lib().hn_weights_rbf_set_variant(0)
    # apply timing, cold L2 and warm
    f = L.to_device(np.sin(ns.positions[:, 0]))
    out = L.empty((3, len(ns)), t.float64)
    rows_d = L.to_device(rows.astype(np.int32))
    for cold in (True, False):
        ts = []
        for rep in range(6):
            if cold:
                flush.fill_(rep)
            e0.record()
            L.call("hn_apply_ell", 1, L.host_i64([K]), L.host_ints([12]), L.host_ptrs([rows_d]), L.host_ptrs([oi]),
                   L.host_ptrs([ow]), 3, L.host_ints([0, 1, 2]), L.ptr(f), L.ptr(out), len(ns), L.stream_handle())
            e1.record()
            t.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts[1:]))
        byt = 28 * K * 12 + 8 * len(ns) + 24 * K
        print(f"apply3 {'cold' if cold else 'warm'}: {ms * 1e3:.1f} us -> {byt / ms / 1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
