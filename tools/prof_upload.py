"""Host cost of the node-set upload variants on this box (dev tool)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402


def main():
    t = L.torch()
    ns = nodesets.jittered_box(315, seed=1)
    pos, kind, sp = np.asarray(ns.positions, float), np.asarray(ns.kind, np.int8), np.asarray(ns.spacing, float)

    def staged():
        return L.to_device_many([pos, kind, sp])

    def direct():  # pageable -> device, driver-staged
        return [t.from_numpy(a).to(L.device()) for a in (pos, kind, sp)]

    def pinned_once():
        return [t.from_numpy(a).pin_memory().to(L.device(), non_blocking=True) for a in (pos, kind, sp)]

    for name, fn in (("to_device_many", staged), ("pageable .to", direct), ("pin_memory().to", pinned_once)):
        for _ in range(5):
            fn()
        t.cuda.synchronize()
        ts = []
        for _ in range(30):
            t0 = time.perf_counter()
            fn()
            t.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(f"{name:18s}: {np.median(ts) * 1e3:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
