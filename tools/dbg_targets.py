"""Debug aid: separate targets at grid edges (which phase fails)."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1802_07844_b200 as hs
from paper_1802_07844_b200.configs import make_system
from paper_1802_07844_b200._plan import get_evaluator
from paper_1802_07844_b200.ewald_fourier import prepare_tables
what = int(sys.argv[1])
s, _ = make_system("cfg3", n=3000)
p = hs.EwaldParams(xi=33.28, rc=0.12, M=128, P=24)
g = p.grid(1.0, "half")
tg = np.array([[0.25, np.nextafter(1.0, 0), 0.5]])
lo = np.floor((tg[:, 1] - g.origin[1]) / g.h) - g.P // 2 + 1
print("lo_y", lo, "ny", g.dims[1])
ev = get_evaluator("stresslet", "half", 1.0, p.xi, p.rc, g, s.n, 1, False)
prepare_tables(ev, s, g, None, None)
try:
    u = ev.execute(s.positions, s.g, s.q, targets=tg, what=what)
    print(what, "ok", u[0])
except Exception as e:
    print(what, type(e).__name__, str(e)[:200])
