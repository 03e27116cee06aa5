"""experiments.py (the reference's benchmark harness, ref:bench.py) on the GPU path."""

import json
import math

import numpy as np
import pytest


def test_records_roundtrip(tmp_path):
    from paper_1802_07844_b200.experiments import BenchRecord, write_records
    r = [BenchRecord("breakdown", "stokeslet", "half", 100, 1.0, 7.0, rc=0.6, M=10, P=14,
                     times={"total": 1.5}, errors={"relative": 1e-9})]
    p = tmp_path / "r.csv"
    write_records(r, p)
    head = p.read_text().splitlines()[0].split(",")
    assert head[-2:] == ["t_total", "e_relative"] or "t_total" in head
    assert json.load(open(str(p) + ".json"))["records"] == 1


@pytest.mark.gpu
def test_break_even_and_breakdown_gpu(gpu):
    from paper_1802_07844_b200.experiments import break_even, runtime_breakdown
    recs, cross = break_even("stokeslet", "half", N_values=(1000, 4000), reps=1)
    assert len(recs) == 2 and all(r.times["total"] > 0 and r.times["direct"] > 0 for r in recs)
    assert cross is None or cross > 0
    br = runtime_breakdown("rotlet", "half", N_values=(4000,), reps=1)
    t = br[0].times
    assert t["total"] > 0 and all(k in t for k in ("gridding", "fft", "scale", "ifft", "gather", "real"))


@pytest.mark.gpu
def test_error_sweeps_follow_estimates(gpu):
    """Fourier error falls with M and real-space error with r_c, tracking the estimates
    (the reference's own sweep semantics)."""
    from paper_1802_07844_b200.experiments import sweep_fourier_error, sweep_real_error
    f = sweep_fourier_error("stokeslet", 800, 1.0, 10.0, (12, 20, 28), max_targets=200)
    rel = [r.errors["relative"] for r in f]
    assert rel[0] > rel[1] > rel[2]
    for r in f:   # the estimate is an RMS bound within a modest factor
        assert r.errors["relative"] < 30 * r.errors["estimate_relative"] + 1e-14
    rr = sweep_real_error("stokeslet", 800, 1.0, 10.0, (0.1, 0.2, 0.3), max_targets=200)
    rel = [r.errors["relative"] for r in rr]
    assert rel[0] > rel[1] > rel[2]
