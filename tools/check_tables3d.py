"""Compare 3D weight tables (interior n=20/30, boundary partial n=30, normal derivative) of
the RBF kernel variants against the CPU oracle on a small sphere set (dev tool)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L  # noqa: E402
from paper_2303_01760_b200 import nodesets  # noqa: E402
from oracle import hn_oracle as O  # noqa: E402


def rel(a, b):
    den = np.maximum(np.abs(b).max(axis=-1), 1e-300)
    return float((np.abs(a - b).max(axis=-1) / den).max())


def main():
    ns = nodesets.hybrid_sphere_3d(int(sys.argv[1]) if len(sys.argv) > 1 else 24, seed=4, refine=2.8)
    b = np.nonzero(ns.boundary_mask)[0]
    print("N", len(ns), "boundary", len(b))
    for v in (100, 0):
        L.lib().hn_weights_rbf_set_variant(v)
        tp = hn.boundary_partial_table(ns, b, exclude=ns.boundary_mask)
        tn = hn.normal_derivative_table(ns, b)
        ti = hn.compute_weights(ns, [hn.Laplacian(), hn.Partial(0), hn.Partial(1), hn.Partial(2)], rbf_n=20)
        for name, t in (("partial", tp), ("normal", tn), ("interior20", ti)):
            for op, w in t.weights.items():
                rows = np.nonzero(t.sizes)[0]
                print(f"variant {v} {name} {op}: finite {np.isfinite(w).all()} maxabs {np.abs(w).max():.3e}")
        if v == 100:
            base = (tp, tn, ti)
        else:
            for name, t, t0 in zip(("partial", "normal", "interior20"), (tp, tn, ti), base):
                assert np.array_equal(t.indices, t0.indices), name
                for op in t.weights:
                    print(f"  {name} {op}: rowwise rel vs searching {rel(t.weights[op], t0.weights[op]):.2e}")
    L.lib().hn_weights_rbf_set_variant(0)


if __name__ == "__main__":
    main()
