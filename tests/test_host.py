"""CPU-only tests: host mirror logic, the C-ABI library surface, seeded workloads."""

import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def test_gridspec_known_answers():
    # test_ewald_fourier.py:22-31 of the reference
    from paper_1802_07844_b200 import GridSpec
    g = GridSpec(L=3.0, M=30, P=16, xi=4.0, geometry="half")
    assert g.h == pytest.approx(0.1)
    assert g.Mtilde == 46
    assert g.Ltilde == pytest.approx(4.6)
    assert g.k_inf == pytest.approx(math.pi / g.h)
    assert g.dims == (46, 46, 92)
    assert g.R == pytest.approx(math.sqrt(6.0) * 4.6)
    assert all(p >= 2 * d for p, d in zip(g.padded_dims, g.dims))
    assert 0.0 < g.eta < 1.0


def test_gridspec_headline():
    from paper_1802_07844_b200 import GridSpec
    g = GridSpec(L=1.0, M=192, P=24, xi=49.92)
    assert g.dims == (216, 216, 432)
    assert g.padded_dims == (480, 480, 924)
    assert g.guard == 24


def test_gridspec_parity_and_validation():
    from paper_1802_07844_b200 import GeometryError, GridSpec, ParameterError
    with pytest.warns(UserWarning):
        g = GridSpec(L=2.0, M=15, P=16, xi=3.0, geometry="free")
    assert (g.M + g.P) % 2 == 0
    with pytest.raises(ParameterError):
        GridSpec(L=-1.0, M=16, P=8, xi=3.0)
    with pytest.raises(GeometryError):
        GridSpec(L=1.0, M=16, P=8, xi=3.0, geometry="periodic")


def test_next_fast_len_matches_scipy():
    import scipy.fft as sfft
    from paper_1802_07844_b200.ewald_fourier import next_fast_len
    for n in list(range(1, 3000)) + [4097, 9999, 123457]:
        assert next_fast_len(n) == sfft.next_fast_len(n), n


def test_gridspec_matches_oracle_grid(oracle):
    from paper_1802_07844_b200 import GridSpec
    for L, M, P, xi, geom in ((1.0, 64, 24, 12.0, "half"), (2.0, 384, 24, 49.92, "half"), (1.0, 33, 16, 7.0, "free")):
        a = GridSpec(L=L, M=M, P=P, xi=xi, geometry=geom)
        b = oracle.Grid(L, M, P, xi, geom)
        assert a.padded_dims == b.padded_dims and a.dims == b.dims and a.guards == b.guards
        assert a.eta == b.eta and a.R == b.R
        np.testing.assert_array_equal(a.origin, b.origin)


def test_table_kinds_and_truncated_hat():
    from paper_1802_07844_b200 import BIHARMONIC, HARMONIC, table_kinds_for, truncated_greens_hat
    assert table_kinds_for("stokeslet", "free") == [BIHARMONIC]
    assert set(table_kinds_for("stokeslet", "half")) == {BIHARMONIC, HARMONIC}
    assert table_kinds_for("rotlet", "free") == [HARMONIC]
    R = 1.7
    assert truncated_greens_hat(HARMONIC, R, np.array([1e-8]))[0] == pytest.approx(2 * math.pi * R**2, rel=1e-10)
    ks = np.array([0.3 - 1e-9, 0.3 + 1e-9]) / 1.3
    v = truncated_greens_hat(BIHARMONIC, 1.3, ks)
    assert abs(v[0] - v[1]) < 1e-8 * abs(v[0])


def test_table_cache_roundtrip(tmp_path):
    from paper_1802_07844_b200 import GreensTable, HARMONIC, load_table, save_table
    rng = np.random.default_rng(0)
    t = GreensTable(kind=HARMONIC, R=2.5, Ltilde=1.2, dims=(4, 6, 8), samples=rng.normal(size=(4, 6, 8)))
    p = tmp_path / "t.segt"
    save_table(t, p)
    with open(p, "rb") as fh:
        assert fh.read(4) == b"SEGT"
    b = load_table(p)
    assert b.kind == HARMONIC and tuple(b.dims) == (4, 6, 8)
    np.testing.assert_array_equal(b.samples, t.samples)


def test_point_system_validation():
    from paper_1802_07844_b200 import GeometryError, ParameterError, PointSystem
    with pytest.raises(ParameterError):
        PointSystem(kind="stokeslet", geometry="half", box_length=1.0, positions=[[0.5, 0.5, 1.0]], f=[[1, 0, 0]])
    with pytest.raises(GeometryError):
        PointSystem(kind="stokeslet", geometry="half", box_length=1.0, positions=[[0.5, 0.5, 0.0]], f=[[1, 0, 0]])


def test_reflect_involution():
    from paper_1802_07844_b200 import generate_system, reflect
    s = generate_system(20, 1.0, "stresslet", "half", seed=1)
    img = reflect(s)
    np.testing.assert_array_equal(img.combined_positions[20:] * [1, 1, -1], s.positions)
    np.testing.assert_array_equal(img.combined_sign, np.r_[np.ones(20), -np.ones(20)])


def test_workloads_match_baseline_shapes():
    from paper_1802_07844_b200.configs import make_system
    s, t = make_system("cfg1")
    assert s.n == 1000 and t is None
    assert s.positions[:, 2].min() >= 0.01 and s.positions.max() < 1.0
    s4, _ = make_system("cfg4", n=50_000)
    assert s4.positions[:, 2].min() >= 0.005 and s4.positions[:, 2].max() < 1.0
    tau = np.cross(s4.g, s4.q)
    assert np.all(np.isfinite(tau))
    s3, _ = make_system("cfg3", n=1000)
    np.testing.assert_allclose(np.linalg.norm(s3.q, axis=1), 1.0)
    s5, t5 = make_system("cfg5", n=1000)
    assert t5.shape == (1000, 3) and s5.box_length == 2.0 and s5.kind == "mixed"
    assert s5.stokeslet.f.shape == (1000, 3) and np.allclose(np.linalg.norm(s5.stresslet.q, axis=1), 1.0)
    f, gq = s5.strengths()
    assert gq.shape == (1000, 6) and np.array_equal(gq[:, :3], s5.stresslet.g)


def test_golden_fixtures_present():
    for name in ("cell_lists", "real_space", "gridding", "tables", "fourier", "ewald", "direct"):
        assert os.path.exists(os.path.join(ROOT, "tests", "golden", name + ".npz"))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "hsewald_b200.h")).read()
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", txt)))


def test_c_abi_exports_every_header_symbol():
    """The built library loads without a GPU and exports every entry point of include/*.h."""
    import ctypes
    from paper_1802_07844_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(_lib.EXPORTED) == set(syms)


def test_no_cpu_fallback_without_device():
    """Without a GPU the product path fails loudly instead of computing on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1802_07844_b200 import DeviceError, EwaldParams, ewald_sum, generate_system
    from paper_1802_07844_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    s = generate_system(10, 1.0, "stokeslet", "half", seed=0)
    with pytest.raises(DeviceError):
        ewald_sum(s, EwaldParams(xi=4.0, rc=0.3, M=16, P=8))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1802_07844_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "hsoracle", "liboracle"):
                    assert bad not in txt, (f, bad)


def test_install_as_hsewald_aliases_reference_modules():
    """Callers written for the reference import it by name; the alias maps them here."""
    import importlib
    import sys
    from paper_1802_07844_b200 import compat, experiments, ewald
    saved = {k: v for k, v in sys.modules.items() if k == "hsewald" or k.startswith("hsewald.")}
    for k in saved:
        del sys.modules[k]
    try:
        compat.install_as_hsewald()
        hsewald = importlib.import_module("hsewald")
        from hsewald.ewald import ewald_sum, EwaldParams  # noqa: F401
        from hsewald.ewald_fourier import GridSpec, get_tables  # noqa: F401
        from hsewald.estimates import select_parameters  # noqa: F401
        assert ewald_sum is ewald.ewald_sum
        assert hsewald.bench is experiments and callable(hsewald.bench.break_even)
        assert hsewald.stokeslet is not None and hsewald.kernel_real is not None
    finally:
        for k in [k for k in sys.modules if k == "hsewald" or k.startswith("hsewald.")]:
            del sys.modules[k]
        sys.modules.update(saved)
