"""Host-side profile of the public-API (e2e) compute_weights call on config 1 (dev tool)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402
from paper_2303_01760_b200.nodegen import NodeSet  # noqa: E402


def call(ns, ops):
    fresh = NodeSet(ns.positions, ns.spacing, ns.kind, ns.role, ns.bc_value, ns.normals, ns.origin, ns.lattice,
                    ns.lattice_idx)
    table = hn.compute_weights(fresh, ops)
    return table.indices, table.weights, table.method


def main():
    t = L.torch()
    ns = nodesets.jittered_box(315, seed=1)
    ops = [hn.Laplacian(), hn.Partial(0), hn.Partial(1)]
    for _ in range(3):
        call(ns, ops)
    t.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        call(ns, ops)
    print(f"e2e call {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        call(ns, ops)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(16)


if __name__ == "__main__":
    main()
