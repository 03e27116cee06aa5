"""estimates.py (host mirror of ref:estimates.py) against golden values produced by the
reference itself (tests/golden/make_estimates_golden.py)."""

import math

import numpy as np
import pytest

from conftest import golden

KINDS = ("stokeslet", "stresslet", "rotlet")
GEOMS = ("free", "half")


def test_estimates_match_reference():
    from paper_1802_07844_b200 import estimates as E
    d = golden("estimates")
    for ki, Q, xi, L, k_inf, R, rc, ef, er in d["est"]:
        kind = KINDS[int(ki)]
        assert math.isclose(E.fourier_truncation_estimate(kind, Q, xi, k_inf, L, R), ef, rel_tol=1e-12, abs_tol=0)
        assert math.isclose(E.real_truncation_estimate(kind, Q, xi, rc, L), er, rel_tol=1e-12, abs_tol=0)


def test_kernel_Q_matches_reference():
    from paper_1802_07844_b200 import estimates as E
    from paper_1802_07844_b200.system import generate_system
    for ki, gi, q in golden("estimates")["q"]:
        s = generate_system(500, 1.3, KINDS[int(ki)], GEOMS[int(gi)], seed=11 + int(ki))
        assert math.isclose(E.kernel_Q(s), q, rel_tol=1e-13)


def test_parameter_selection_matches_reference():
    from paper_1802_07844_b200 import estimates as E
    for ki, gi, tol, xi, Q, rc, M in golden("estimates")["sel"]:
        kind, geom = KINDS[int(ki)], GEOMS[int(gi)]
        if rc < 0:
            with pytest.raises(E.InfeasibleToleranceError):
                E.select_rc(kind, tol, xi, 1.3, Q)
        else:
            assert math.isclose(E.select_rc(kind, tol, xi, 1.3, Q), rc, rel_tol=1e-12)
        if M < 0:
            with pytest.raises(E.InfeasibleToleranceError):
                E.select_M(kind, tol, xi, 1.3, Q, geom, P=24)
        else:
            assert E.select_M(kind, tol, xi, 1.3, Q, geom, P=24) == int(M)


def test_eta_guard_and_errors():
    from paper_1802_07844_b200 import estimates as E
    from paper_1802_07844_b200.errors import ParameterError
    # large xi at small M gives eta >= 1: the guarded scan moves to a finer grid
    M0 = E.select_M("stokeslet", 1e-3, 40.0, 1.0, 1.0, "half", P=24)
    M1 = E.select_M("stokeslet", 1e-3, 40.0, 1.0, 1.0, "half", P=24, eta_guard=True)
    assert M1 >= M0 and E.grid_eta(M1, 24, 40.0, 1.0) < 1.0
    with pytest.raises(ParameterError):
        E.real_truncation_estimate("stokeslet", 1.0, -1.0, 0.1, 1.0)
    m = E.measure_error(np.ones((4, 3)), 2 * np.ones((4, 3)))
    assert math.isclose(m.relative, 0.5)
