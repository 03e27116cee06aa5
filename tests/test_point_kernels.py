"""Single-point kernel helpers (point_kernels.py) vs golden values made by the reference."""

import numpy as np
import pytest

from conftest import golden

KINDS = ("stokeslet", "stresslet", "rotlet")


def test_point_kernels_match_reference():
    import paper_1802_07844_b200 as hs
    from paper_1802_07844_b200 import kernels_direct as K
    from paper_1802_07844_b200 import ewald_real as R
    d = golden("point_kernels")
    r, g, q, f, y, x = d["r"], d["g"], d["q"], d["f"], d["y"], d["x"]
    n = r.shape[0]
    close = lambda a, b: np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-13 * np.max(np.abs(b)))  # noqa: E731
    close(np.array([hs.stokeslet(a) for a in r]), d["stokeslet"])
    close(np.array([hs.stresslet_apply(a, b, c) for a, b, c in zip(r, g, q)]), d["stresslet_apply"])
    close(np.array([K.rotlet_apply(a, b, c) for a, b, c in zip(r, g, q)]), d["rotlet_apply"])
    hd = [hs.harmonic_derivs(a) for a in r]
    close(np.array([h.G for h in hd]), d["hd_G"])
    close(np.array([h.gradG for h in hd]), d["hd_grad"])
    close(np.array([h.hessG for h in hd]), d["hd_hess"])
    close(np.array([h.thirdG for h in hd]), d["hd_third"])
    for kind in KINDS:
        kw = lambda i: ({"f": f[i]} if kind == "stokeslet" else {"g": g[i], "q": q[i]})  # noqa: E731
        ph = [hs.correction_phi(kind, y[i], x[i], **kw(i)) for i in range(n)]
        close(np.array([p[0] for p in ph]), d[f"cphi_{kind}"])
        close(np.array([p[1] for p in ph]), d[f"cgrad_{kind}"])
        close(np.array([R.kernel_real(kind, r[i], 7.5) for i in range(n)]), d[f"kreal_{kind}"])
    close(np.array(hs.f_derivs(np.abs(r[:, 0]) + 0.01, 7.5)), d["f_derivs"])


def test_point_kernels_singular():
    import paper_1802_07844_b200 as hs
    with pytest.raises(hs.SingularityError):
        hs.stokeslet([0.0, 0.0, 0.0])
    with pytest.raises(hs.SingularityError):
        hs.correction_phi("stokeslet", [0.1, 0.2, 0.3], [0.1, 0.2, -0.3], f=[1.0, 0.0, 0.0])
