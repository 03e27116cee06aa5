"""One free-space evaluation of the HL-sized system (3 spread channels); prints the phase times.
Used to A/B spread variants whose register need depends on the channel count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_07844_b200 import GridSpec  # noqa: E402
from paper_1802_07844_b200._plan import Evaluator  # noqa: E402
from paper_1802_07844_b200.configs import WORKLOADS, make_system  # noqa: E402

w = WORKLOADS["HL"]
s, tg = make_system(w)
grid = GridSpec(L=w.L, M=w.M, P=w.P, xi=w.xi, geometry="free")
ev = Evaluator(w.kind, "free", w.L, w.xi, w.rc, grid, s.n, s.n, True)
ev.build_tables()
pos, sa = torch.from_numpy(s.positions).cuda(), torch.from_numpy(s.f).cuda()
for i in range(4):
    u, ur, uf, t = ev.execute(pos, sa, None, what=7)  # bit 2: pipelines serialised (per-phase times)
torch.cuda.synchronize()
print({k: round(v, 3) for k, v in t.items()})
