"""Golden values of the reference's single-point kernel helpers (ref:kernels_direct.py,
ref:ewald_real.py), made by importing the REFERENCE in the build container:
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_point_kernel_golden.py
Writes tests/golden/point_kernels.npz."""

import os

import numpy as np

from hsewald import ewald_real as R  # noqa: E402  (the reference, from PYTHONPATH)
from hsewald import kernels_direct as K  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(31)
n = 12
r = rng.normal(size=(n, 3)) * 0.3
g, q, f = rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), rng.normal(size=(n, 3))
y = np.column_stack([rng.uniform(0, 1, (n, 2)), rng.uniform(0.05, 1, n)])
x = np.column_stack([rng.uniform(0, 1, (n, 2)), rng.uniform(0.0, 1, n)])
out = {"r": r, "g": g, "q": q, "f": f, "y": y, "x": x}
out["stokeslet"] = np.array([K.stokeslet(a) for a in r])
out["stresslet_apply"] = np.array([K.stresslet_apply(a, b, c) for a, b, c in zip(r, g, q)])
out["rotlet_apply"] = np.array([K.rotlet_apply(a, b, c) for a, b, c in zip(r, g, q)])
hd = [K.harmonic_derivs(a) for a in r]
out["hd_G"] = np.array([h.G for h in hd])
out["hd_grad"] = np.array([h.gradG for h in hd])
out["hd_hess"] = np.array([h.hessG for h in hd])
out["hd_third"] = np.array([h.thirdG for h in hd])
for kind in ("stokeslet", "stresslet", "rotlet"):
    kw = lambda i: ({"f": f[i]} if kind == "stokeslet" else {"g": g[i], "q": q[i]})  # noqa: E731
    ph = [K.correction_phi(kind, y[i], x[i], **kw(i)) for i in range(n)]
    out[f"cphi_{kind}"] = np.array([p[0] for p in ph])
    out[f"cgrad_{kind}"] = np.array([p[1] for p in ph])
    out[f"kreal_{kind}"] = np.array([R.kernel_real(kind, r[i], 7.5) for i in range(n)])
fd = R.f_derivs(np.abs(r[:, 0]) + 0.01, 7.5)
out["f_derivs"] = np.array(fd)
np.savez(os.path.join(HERE, "point_kernels.npz"), **out)
print("ok", len(out))
