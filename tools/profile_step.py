"""One headline (HL) evaluation for profiling: builds the plan + tables, runs
`--iters` evaluations with device-resident inputs.  Used under ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1802_07844_b200 import GridSpec  # noqa: E402
from paper_1802_07844_b200._plan import Evaluator  # noqa: E402
from paper_1802_07844_b200.configs import WORKLOADS, make_system  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="HL")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
w = WORKLOADS[a.workload]
s, tg = make_system(w, n=a.n)
grid = GridSpec(L=w.L, M=w.M, P=w.P, xi=w.xi)
nt = s.n if tg is None else tg.shape[0]
ev = Evaluator(w.kind, "half", w.L, w.xi, w.rc, grid, s.n, nt, tg is None)
ev.build_tables()
from paper_1802_07844_b200.ewald import _strengths  # noqa: E402
fa, fb = _strengths(s)
put = lambda x: None if x is None else torch.from_numpy(x).cuda()  # noqa: E731
pos, sa, sb, tgd = put(s.positions), put(fa), put(fb), put(tg)
for i in range(a.iters):
    u, ur, uf, t = ev.execute(pos, sa, sb, targets=tgd)
torch.cuda.synchronize()
print({k: round(v, 3) for k, v in t.items()})
