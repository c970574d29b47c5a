"""Time the MON weight kernel (2D config-2 rows, 3D config-4 rows) and check it against the
general-path build via HN_LIB_PATH A/B (dev tool): prints time and a weight checksum."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402
from paper_2303_01760_b200._device import device_nodes  # noqa: E402


def main():
    t = L.torch()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    flush = L.empty(64 * 2 ** 20, t.float64)
    out = Path(__file__).resolve().parents[1] / "gpurun_out"
    for name, ns, nops in (("2D config2", nodesets.hybrid_hole_2d(500, seed=2), 3),
                           ("3D config4", nodesets.hybrid_sphere_3d(94, seed=4, refine=2.8), 4)):
        dn = device_nodes(ns)
        d = ns.dim
        method = dn.classify().cpu().numpy()
        rows = np.nonzero(method == 0)[0].astype(np.int32)
        st = dn.mon_stencils(L.to_device(rows))
        K, n = int(st.shape[0]), int(st.shape[1])
        kinds = L.host_ints([0] + [1] * d)
        axes = L.host_ints([0] + list(range(d)))
        nrm = L.host_dbls([0.0] * (nops * d))
        oi = L.empty((n, K), t.int32)
        ow = L.empty((nops, n, K), t.float64)
        info = L.zeros(K, t.int32)
        ts = []
        for rep in range(6):
            flush.fill_(rep)
            e0.record()
            L.call("hn_weights_mon", L.ptr(dn.pos), d, L.ptr(st), K, nops, kinds, axes, nrm, L.ptr(oi), L.ptr(ow),
                   L.ptr(info), L.stream_handle())
            e1.record()
            t.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        w = ow.cpu().numpy()
        f = out / f"mon_{d}d.npy"
        if f.exists():
            ref = np.load(f)
            rel = (np.abs(w - ref).max(axis=(0, 1)) / np.maximum(np.abs(ref).max(axis=(0, 1)), 1e-300)).max()
            cmp = f"max row rel diff vs saved {rel:.2e}"
        else:
            np.save(f, w)
            cmp = "saved"
        print(f"{name}: {K} MON stencils, {np.median(ts[1:]) * 1e3:.1f} us, idx equal: "
              f"{bool((oi.cpu().numpy() >= 0).all())}, singular {int((info != 0).sum().item())}, {cmp}", flush=True)


if __name__ == "__main__":
    main()
