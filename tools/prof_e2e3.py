"""Host-time breakdown of the public-API compute_weights call (dev tool): wraps the main
stages with perf_counter accumulators (no extra synchronisation is added)."""
import sys
import time
from collections import defaultdict
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _device, _lib as L, approx, nodegen, nodesets  # noqa: E402

ACC = defaultdict(float)
CNT = defaultdict(int)


def wrap(owner, name, label=None):
    fn = getattr(owner, name)
    label = label or f"{getattr(owner, '__name__', owner)}.{name}"

    def inner(*a, **k):
        t0 = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            ACC[label] += time.perf_counter() - t0
            CNT[label] += 1
    setattr(owner, name, inner)


def main():
    t = L.torch()
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    ns = {1: lambda: nodesets.jittered_box(315, seed=1), 2: lambda: nodesets.hybrid_hole_2d(500, seed=2),
          4: lambda: nodesets.hybrid_sphere_3d(94, seed=4, refine=2.8)}[cfg]()
    dim = ns.dim
    ops = [hn.Laplacian()] + [hn.Partial(a) for a in range(dim)]
    rbf_n = 20 if dim == 3 else None

    def call():
        fresh = nodegen.NodeSet(ns.positions, ns.spacing, ns.kind, ns.role, ns.bc_value, ns.normals, ns.origin,
                                ns.lattice, ns.lattice_idx)
        tab = hn.compute_weights(fresh, ops, rbf_n=rbf_n)
        return tab.indices, tab.weights

    for _ in range(3):
        call()
    t.cuda.synchronize()
    reps = 10
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    t.cuda.synchronize()
    print(f"config {cfg}: e2e call {(time.perf_counter() - t0) / reps * 1e3:.3f} ms (unwrapped)", flush=True)

    wrap(_device.DeviceNodes, "__init__", "DeviceNodes.__init__")
    wrap(_device.DeviceNodes, "grid", "DeviceNodes.grid")
    wrap(_device.DeviceNodes, "knn", "DeviceNodes.knn")
    wrap(_device.DeviceNodes, "classify", "DeviceNodes.classify")
    wrap(_device.DeviceTable, "host_arrays", "DeviceTable.host_arrays")
    wrap(approx, "_check_info")
    wrap(approx, "_solve_bin")
    wrap(approx, "_interior_device_table")
    wrap(L, "to_device")
    wrap(L, "call")
    orig_call = L.call

    def named_call(name, *a):
        t0 = time.perf_counter()
        try:
            return orig_call(name, *a)
        finally:
            ACC["  call:" + name] += time.perf_counter() - t0
            CNT["  call:" + name] += 1
    L.call = named_call
    wrap(nodegen.NodeSet, "__init__", "NodeSet.__init__")
    ACC.clear()
    CNT.clear()
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    t.cuda.synchronize()
    print(f"wrapped e2e call {(time.perf_counter() - t0) / reps * 1e3:.3f} ms", flush=True)
    for k, v in sorted(ACC.items(), key=lambda kv: -kv[1]):
        print(f"  {1e3 * v / reps:8.3f} ms/call  x{CNT[k] / reps:4.1f}  {k}")


if __name__ == "__main__":
    main()
