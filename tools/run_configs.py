"""Time every BASELINE workload (one evaluation after warm-up) and check accuracy on a
target subset against the GPU direct sum.  Output: one JSON line per workload."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1802_07844_b200 as hs  # noqa: E402
from paper_1802_07844_b200._plan import Evaluator  # noqa: E402
from paper_1802_07844_b200.configs import WORKLOADS, make_system  # noqa: E402

names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "HL", "cfg5"]
for name in names:
    w = WORKLOADS[name]
    s, tg = make_system(w)
    grid = hs.GridSpec(L=w.L, M=w.M, P=w.P, xi=w.xi)
    nt = s.n if tg is None else tg.shape[0]
    ev = Evaluator(w.kind, "half", w.L, w.xi, w.rc, grid, s.n, nt, tg is None)
    t0 = time.perf_counter()
    ev.build_tables()
    t_tab = time.perf_counter() - t0
    dev = torch.device("cuda")
    pos = torch.from_numpy(s.positions).to(dev)
    from paper_1802_07844_b200.ewald import _strengths
    fa, fb = _strengths(s)
    sa = torch.from_numpy(np.ascontiguousarray(fa)).to(dev)
    sb = None if fb is None else torch.from_numpy(np.ascontiguousarray(fb)).to(dev)
    tgd = None if tg is None else torch.from_numpy(tg).to(dev)
    for _ in range(2):
        u, ur, uf, t = ev.execute(pos, sa, sb, targets=tgd)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        u, ur, uf, t = ev.execute(pos, sa, sb, targets=tgd)
        times.append(t)
    torch.cuda.synchronize()
    tm = {k: float(np.median([x[k] for x in times])) for k in times[0]}
    u = u.cpu().numpy()
    sub = np.arange(0, nt, max(1, nt // 300))
    if tg is None:
        ud = hs.direct_sum_half(s, targets=s.positions[sub], target_indices=sub).velocities
    else:
        ud = hs.direct_sum_half(s, targets=tg[sub]).velocities
    err = float(np.linalg.norm(u[sub] - ud) / np.linalg.norm(ud))
    print(json.dumps({"workload": name, "kind": w.kind, "n": s.n, "n_targets": nt, "M": grid.M, "xi": w.xi,
                      "rc": w.rc, "padded": list(grid.padded_dims), "ms_total": tm["total"],
                      "target_evals_per_s": nt / (tm["total"] * 1e-3),
                      "phases_ms": {k: round(tm[k], 3) for k in ("real", "gridding", "fft", "scale", "ifft", "gather")},
                      "pairs": tm["pairs"], "image_pairs": tm["image_pairs"], "tables_s": round(t_tab, 3),
                      "plan_GB": round(ev.device_bytes / 1e9, 2), "rel_l2_vs_direct_subset": err}), flush=True)
    del ev
    torch.cuda.empty_cache()
