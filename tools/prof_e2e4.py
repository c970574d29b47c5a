"""Host timeline of one public-API compute_weights call on config 1 (dev tool): every libhn
call, torch op site and synchronisation with its host timestamp, to find host-bound gaps."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _device, _lib as L, approx, nodegen, nodesets  # noqa: E402

EV = []


def main():
    t = L.torch()
    ns = nodesets.jittered_box(315, seed=1)
    ops = [hn.Laplacian(), hn.Partial(0), hn.Partial(1)]

    def call():
        fresh = nodegen.NodeSet(ns.positions, ns.spacing, ns.kind, ns.role, ns.bc_value, ns.normals, ns.origin,
                                ns.lattice, ns.lattice_idx)
        t.cuda.synchronize()
        EV.clear()
        EV.append(("start", time.perf_counter()))
        tab = hn.compute_weights(fresh, ops)
        a, b = tab.indices, tab.weights
        EV.append(("end", time.perf_counter()))
        return a, b

    for _ in range(5):
        call()
    orig = L.call

    def traced(name, *a):
        t0 = time.perf_counter()
        r = orig(name, *a)
        EV.append((name, t0, time.perf_counter()))
        return r
    L.call = traced
    orig_sync = t.cuda.Stream.synchronize

    def tsync(self):
        t0 = time.perf_counter()
        r = orig_sync(self)
        EV.append(("stream.synchronize", t0, time.perf_counter()))
        return r
    t.cuda.Stream.synchronize = tsync
    orig_cpu = t.Tensor.cpu

    def tcpu(self, *a, **k):
        t0 = time.perf_counter()
        r = orig_cpu(self, *a, **k)
        EV.append((f"tensor.cpu {tuple(self.shape)}", t0, time.perf_counter()))
        return r
    t.Tensor.cpu = tcpu
    for _ in range(3):
        call()
    t0 = EV[0][1]
    for e in EV:  # timeline of the last traced call
        if len(e) == 2:
            print(f"{(e[1] - t0) * 1e3:8.3f} ms  {e[0]}")
        else:
            print(f"{(e[1] - t0) * 1e3:8.3f} ms  +{(e[2] - e[1]) * 1e3:6.3f}  {e[0]}")
    # plain timing for several chunk counts of the native pipeline
    t.cuda.Stream.synchronize = orig_sync
    t.Tensor.cpu = orig_cpu
    L.call = orig
    for ch in (1, 2, 4, 8):
        approx.NATIVE_CHUNKS = ch
        for _ in range(3):
            call()
        ts = []
        for _ in range(10):
            call()
            ts.append(EV[-1][1] - EV[0][1])
        print(f"chunks {ch}: e2e {np.median(ts) * 1e3:.3f} ms")
    approx.NATIVE_CHUNKS = 8
    t0 = EV[0][1]
    for e in EV:
        if len(e) == 2:
            print(f"{(e[1] - t0) * 1e3:8.3f} ms  {e[0]}")
        else:
            print(f"{(e[1] - t0) * 1e3:8.3f} ms  +{(e[2] - e[1]) * 1e3:6.3f}  {e[0]}")


if __name__ == "__main__":
    main()
