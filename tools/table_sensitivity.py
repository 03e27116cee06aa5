"""Where the GPU-vs-oracle difference at a full-size configuration comes from: the Green's
tables (both are round-off-level restatements of ref:ewald_fourier.py:207-244) or the evaluation.
(1) GPU precompute_greens vs the oracle's precompute_greens_half on the same grid;
(2) the GPU evaluation with the ORACLE's tables (tables=) and with its own, both against the
fixture tests/golden/fullsize_<cfg>.npz.  Usage: python tools/table_sensitivity.py cfg5"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1802_07844_b200 as hs  # noqa: E402
from oracle import hsoracle as H  # noqa: E402
from paper_1802_07844_b200 import _plan  # noqa: E402
from paper_1802_07844_b200.configs import WORKLOADS, make_system  # noqa: E402
from paper_1802_07844_b200.ewald import ewald_sum_mixed  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
w = WORKLOADS[name]
s, tg = make_system(w)
d = np.load(os.path.join("tests", "golden", f"fullsize_{name}.npz"))
idx = d["idx"]
p = hs.EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P)
grid = p.grid(w.L, "half")
go = H.Grid(w.L, w.M, w.P, w.xi)
H.set_threads(os.cpu_count())
kinds = ["biharmonic", "harmonic"] if w.kind != "rotlet" else ["harmonic"]
out = {"workload": name}
otab = {}
for k in kinds:
    half = H.precompute_greens_half(k, go, workers=os.cpu_count())
    gt = hs.precompute_greens(k, grid, max_bytes=None).samples[..., : half.shape[2]]
    diff = np.abs(gt - half)
    out[f"{k}_max_abs_diff_rel_to_max"] = float(diff.max() / np.abs(half).max())
    out[f"{k}_rel_l2"] = float(np.linalg.norm(gt - half) / np.linalg.norm(half))
    del gt
    otab[k] = hs.GreensTable(kind=k, R=grid.R, Ltilde=grid.Ltilde, dims=tuple(grid.padded_dims),
                             samples=H.expand_half_table(half, grid.padded_dims))
    del half
ev = ewald_sum_mixed if w.kind == "mixed" else hs.ewald_sum
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
for label, tabs in (("gpu_tables", None), ("oracle_tables", otab)):
    _plan.clear_cache()
    r = ev(s, p, tables=tabs, targets=tg) if tg is not None else ev(s, p, tables=tabs)
    out[label] = {"u": rel(r.velocities[idx], d["u"]), "fourier": rel(r.parts["fourier"][idx], d["u_fourier"]),
                  "real": rel(r.parts["real"][idx], d["u_real"])}
    print(json.dumps(out), flush=True)
print(json.dumps(out))
