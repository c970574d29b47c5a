"""Golden condition numbers from the REFERENCE itself (test infrastructure).

Usage (in the build container, where /root/reference exists):
    OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 python oracle/make_golden_kappa.py

Loads the committed golden node sets (tests/golden/<case>.npz), runs the reference's
compute_weights(..., with_kappa=True) on them (approx.py:379-413 -> the SVD diagnostics of
approx.py:229-233, 285-289) and writes tests/golden/kappa_<case>.npz (kappa per node and
the method array).  The reference package is imported read-only from /root/reference.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

from make_golden import R_approx, ref_nodeset  # noqa: E402



def load_golden(name):
    from paper_2303_01760_b200.nodegen import NodeSet
    with np.load(ROOT / "tests" / "golden" / f"{name}.npz", allow_pickle=False) as z:
        data = {k: z[k] for k in z.files}
    return NodeSet.from_arrays({k[3:]: v for k, v in data.items() if k.startswith("ns_")}), data

CASES = ["dvd_coarse", "config1_small", "config2_small", "config4_small"]


def main():
    for case in CASES:
        ns, _ = load_golden(case)
        dim = ns.positions.shape[1]
        ops = [R_approx.Laplacian()] + [R_approx.Partial(a) for a in range(dim)]
        t = R_approx.compute_weights(ref_nodeset(ns), ops, with_kappa=True)
        out = ROOT / "tests" / "golden" / f"kappa_{case}.npz"
        np.savez_compressed(out, kappa=np.asarray(t.kappa, dtype=np.float64), method=np.asarray(t.method))
        fin = np.isfinite(t.kappa)
        print(case, "nodes", len(ns), "finite kappa", int(fin.sum()), "max", float(np.max(t.kappa[fin])), "->", out)


if __name__ == "__main__":
    main()
