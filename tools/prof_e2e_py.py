"""cProfile of the Python host work in one public compute_weights call (config 1; dev tool)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodegen, nodesets  # noqa: E402


def main():
    t = L.torch()
    ns = nodesets.jittered_box(315, seed=1)
    ops = [hn.Laplacian(), hn.Partial(0), hn.Partial(1)]

    def call():
        fresh = nodegen.NodeSet(ns.positions, ns.spacing, ns.kind, ns.role, ns.bc_value, ns.normals, ns.origin,
                                ns.lattice, ns.lattice_idx)
        tab = hn.compute_weights(fresh, ops)
        return tab.indices, tab.weights
    for _ in range(10):
        call()
    t.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        call()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
