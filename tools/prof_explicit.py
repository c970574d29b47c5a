"""Run the explicit part of a Boussinesq step (K7 + K8 + K10 + K11, pressure held) on the
full config-4 (or config-3) node set, for ncu captures and per-kernel timing (dev tool).
  python tools/prof_explicit.py [4|3] [reps]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    t = L.torch()
    ns = bench.build_nodeset(cfg, 0)
    st, _, _ = bench._stepper(hn, ns, False, 1e5 if cfg == 4 else 1e6)
    flush = bench.L2Flush(L)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        flush(1.0)
        e0.record()
        st.explicit_step()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    S = int(sum(b.K * b.width for b in st.ops._table.bins))
    d, n = ns.dim, len(ns)
    nbytes = S * (28 + 24 * d) + 40 * n * (d + 1)
    ms = float(np.median(ts[1:])) if reps > 1 else ts[0]
    print(f"config {cfg}: N={n} S={S} explicit {ms * 1e3:.1f} us -> {nbytes / ms / 1e6:.0f} GB/s "
          f"({nbytes / 1e6:.1f} MB)", flush=True)


if __name__ == "__main__":
    main()
