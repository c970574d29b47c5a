"""Time the with_kappa diagnostic on the GPU (hn_condition_numbers) against the host SVD
on configs 1 and 4 (dev tool)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, approx  # noqa: E402
from paper_2303_01760_b200._device import device_nodes  # noqa: E402


def main():
    t = L.torch()
    for cfg in (1, 4):
        ns = bench.build_nodeset(cfg, 0)
        ops = [hn.Laplacian()] + [hn.Partial(a) for a in range(ns.dim)]
        tab = approx._compute_weights(ns, ops, rbf_n=20 if ns.dim == 3 else None)
        dn = device_nodes(ns)
        for b in tab._device.bins:
            if b.width == 0:
                continue
            mon = b.width == approx.MON_SIZE[ns.dim]
            approx._kappa_bin(dn, b.d_idx, 1, b.K, b.d_rows, b.K, b.width, mon)
            t.cuda.synchronize()
            t0 = time.perf_counter()
            k = approx._kappa_bin(dn, b.d_idx, 1, b.K, b.d_rows, b.K, b.width, mon)
            t.cuda.synchronize()
            dt = time.perf_counter() - t0
            rows = b.rows_host[:2000]
            idx = b.d_idx[:, :2000].cpu().numpy().T
            st = approx._stencil_order(rows, np.sort(idx, axis=1))
            t1 = time.perf_counter()
            ref = approx._kappa_host(ns.positions, st, mon)
            dh = (time.perf_counter() - t1) / len(rows) * b.K
            err = np.max(np.abs(k[:2000].cpu().numpy() - ref) / ref)
            print(f"config {cfg} width {b.width} K={b.K}: GPU {dt * 1e3:.2f} ms, host SVD ~{dh:.1f} s "
                  f"(from 2000), max rel diff {err:.1e}", flush=True)


if __name__ == "__main__":
    main()
