"""Config-3 time steps without CUDA graphs, the pressure solve in the dev-only eager mode
(HN_PRESSURE_EAGER=1: its kernels enqueued directly), so ncu lists every kernel of a step
(ncu does not descend into conditional graph nodes).  Dev tool:
  HN_PRESSURE_EAGER=1 ncu --metrics gpu__time_duration.sum ... python tools/prof_step_eager.py [steps]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HN_PRESSURE_EAGER", "1")
import bench  # noqa: E402
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    ns = bench.build_nodeset(3, 0)
    st, _, _ = bench._stepper(hn, ns, True, 1e6)
    st.graphs_enabled = False
    for _ in range(steps):
        st.step()
    L.torch().cuda.synchronize()
    st.check_finite()
    print("steps", st.steps, "ok", flush=True)


if __name__ == "__main__":
    main()
