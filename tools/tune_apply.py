"""Cold-L2 timing of the fused ELL apply (Lap + grads) on configs 1, 2, 4 for several block
sizes (dev tool)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _device, _lib as L, approx, nodesets  # noqa: E402


def main():
    t = L.torch()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    flush = L.empty(32 << 20, t.float64)
    for name, ns, rbf_n in (("config1", nodesets.jittered_box(315, seed=1), None),
                            ("config2", nodesets.hybrid_hole_2d(500, seed=2), None),
                            ("config4", nodesets.hybrid_sphere_3d(94, seed=4, refine=2.8), 20)):
        ops = [hn.Laplacian()] + [hn.Partial(a) for a in range(ns.dim)]
        dev = approx._interior_device_table(ns, ops, rbf_n)
        nb, K, W, R, I, Wt, live = _device.bins_args(dev.bins)
        f = L.to_device(nodesets.sinusoid_field(ns.positions))
        out = L.empty((len(ops), len(ns)), t.float64)
        sel = L.host_ints(list(range(len(ops))))
        S = int(sum(b.K * b.width for b in live))
        nbytes = (4 + 8 * len(ops)) * S + 8 * len(ns) + 8 * len(ops) * len(ns) + 4 * len(ns)
        ref = None
        for th in (64, 128, 256):
            L.lib().hn_apply_set_threads(th)
            ts = []
            for _ in range(12):
                flush.fill_(1.0)
                e0.record()
                L.call("hn_apply_ell", nb, K, W, R, I, Wt, len(ops), sel, L.ptr(f), L.ptr(out), len(ns),
                       L.stream_handle())
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            o = out.cpu().numpy()
            same = ref is None or np.array_equal(o, ref)
            ref = o if ref is None else ref
            ms = float(np.median(ts[2:]))
            print(f"{name} threads {th}: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s  identical={same}", flush=True)
        L.lib().hn_apply_set_threads(128)


if __name__ == "__main__":
    main()
