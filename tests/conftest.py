import os
import sys
from pathlib import Path

for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(var, "1")

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the libhn.so kernels")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name: str):
    from paper_2303_01760_b200.nodegen import NodeSet

    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        data = {k: z[k] for k in z.files}
    ns = NodeSet.from_arrays({k[3:]: v for k, v in data.items() if k.startswith("ns_")})
    return ns, data


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get


GOLDEN_CASES = ["dvd_coarse", "scattered_cloud", "config0_small_ref", "config0_small", "config1_small",
                "config2_small", "config4_small"]
