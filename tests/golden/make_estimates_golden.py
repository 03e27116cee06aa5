"""Golden values of the reference's estimates module (ref:estimates.py), made by importing
the REFERENCE in the build container:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_estimates_golden.py
Writes tests/golden/estimates.npz."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
from hsewald import estimates as E  # noqa: E402  (the reference, from PYTHONPATH)
from hsewald.system import generate_system  # noqa: E402

KINDS = ("stokeslet", "stresslet", "rotlet")
rows_est, rows_sel, rows_q = [], [], []
rng = np.random.default_rng(77)
for ki, kind in enumerate(KINDS):
    for gi, geom in enumerate(("free", "half")):
        s = generate_system(500, 1.3, kind, geom, seed=11 + ki)
        rows_q.append([ki, gi, E.kernel_Q(s)])
        for _ in range(12):
            Q, xi, L = 10 ** rng.uniform(0, 4), rng.uniform(2, 60), rng.uniform(0.5, 3)
            k_inf, R, rc = rng.uniform(10, 400), rng.uniform(0.5, 8), rng.uniform(0.02, 1.0)
            rows_est.append([ki, Q, xi, L, k_inf, R, rc, E.fourier_truncation_estimate(kind, Q, xi, k_inf, L, R),
                             E.real_truncation_estimate(kind, Q, xi, rc, L)])
        for tol in (1e-4, 1e-8, 1e-10):
            for xi in (7.0, 12.0, 33.28):
                Q = E.kernel_Q(s)
                try:
                    rc = E.select_rc(kind, tol, xi, 1.3, Q)
                except E.InfeasibleToleranceError:
                    rc = -1.0
                try:
                    M = E.select_M(kind, tol, xi, 1.3, Q, geom, P=24)
                except E.InfeasibleToleranceError:
                    M = -1
                rows_sel.append([ki, gi, tol, xi, Q, rc, M])
np.savez(os.path.join(HERE, "estimates.npz"), est=np.array(rows_est), sel=np.array(rows_sel), q=np.array(rows_q))
print(len(rows_est), len(rows_sel))
