"""Small evaluations that exercise every production kernel once, for compute-sanitizer
(tools/sanitize.sh): cell-list sort (multi-CTA scan), pair kernel (all kinds + audit), the
mirrored DMMA spread (mbarrier / cp.async ring), z / y / x FFT stages (register x stage with
cp.async staging), gather (cp.async ring), table precompute, mixed plan, 2-way slab pipeline,
direct sum.  Checks the results against the single-kind references so a run that silently
corrupts memory also fails."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1802_07844_b200 as hs  # noqa: E402
from paper_1802_07844_b200.configs import make_system  # noqa: E402
from paper_1802_07844_b200.ewald import ewald_sum_mixed  # noqa: E402
from paper_1802_07844_b200.sharding import ewald_sum_slab_local  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
p = hs.EwaldParams(xi=33.28, rc=0.12, M=128, P=24)   # padded (352, 352, 660): register x / y stages
out = {}
for name in ("cfg2", "cfg3", "cfg4"):
    s, _ = make_system(name, n=n)
    r = hs.ewald_sum(s, p)
    d = hs.direct_sum_half(s, targets=s.positions[:50], target_indices=np.arange(50)).velocities
    out[name] = float(np.linalg.norm(r.velocities[:50] - d) / np.linalg.norm(d))
s5, tg = make_system("cfg5", n=n)
p5 = hs.EwaldParams(xi=20.8, rc=0.17, M=80, P=24)
rm = ewald_sum_mixed(s5, p5, targets=tg[:2000])
ra = hs.ewald_sum(s5.stokeslet, p5, targets=tg[:2000]).velocities + hs.ewald_sum(s5.stresslet, p5, targets=tg[:2000]).velocities
out["mixed_vs_sum"] = float(np.linalg.norm(rm.velocities - ra) / np.linalg.norm(ra))
s, _ = make_system("cfg2", n=n)
rs = ewald_sum_slab_local(s, p, 2)
out["slab2_vs_single"] = float(np.linalg.norm(rs.velocities - hs.ewald_sum(s, p).velocities) /
                               np.linalg.norm(rs.velocities))
from paper_1802_07844_b200 import _lib  # noqa: E402
if os.environ.get("HSEWALD_CHECKED") == "1":
    out["device_checks"] = _lib.debug_checks()
print(out)
if "device_checks" in out:
    assert out["device_checks"]["failures"] == 0, out["device_checks"]
assert out["mixed_vs_sum"] < 5e-12 and out["slab2_vs_single"] < 1e-12
assert all(out[k] < 1e-6 for k in ("cfg2", "cfg3", "cfg4"))
