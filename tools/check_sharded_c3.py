"""Row-sharded step at config 3 (full N) with R virtual ranks in lockstep on one GPU against the
single-GPU stepper: bitwise comparison of the fields after a few steps, plus the halo sizes
(dev tool / record for profiles/).   python tools/check_sharded_c3.py [ranks=2] [steps=20]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import sharded as S  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ns = bench.build_nodeset(3, 0)
single, ops, dt = bench._stepper(hn, ns, True, 1e6)
st0 = single.state()
tr = S.LocalTransport(world)
ranks = [S.ShardedStepper(ops, single.params, single.settings, dt, st0, r, world, transport=tr) for r in range(world)]
for _ in range(steps):
    single.step()
    S.step_lockstep(ranks, tr)
want = single.state()
got = S.gather_states(ranks, tr)[0]
same = all(a.tobytes() == b.tobytes() for a, b in ((got.velocity, want.velocity), (got.temperature, want.temperature),
                                                   (got.pressure, want.pressure)))
print(f"config 3 N={len(ns)} ranks={world} steps={steps}: fields bitwise equal to the single-GPU stepper: {same}")
for r in ranks:
    print(f"  rank {r.rank}: owned rows {r.plan.n_own}, halo nodes {r.plan.n_halo}, sent per exchange {len(r.plan.send_loc)}")
assert same
