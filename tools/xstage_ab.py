"""Fourier part of a 1e5-source system on the grid of M (192 -> x-stage length 480, 128 -> 352)
with the current x-stage; saves the velocities to argv[1] (compares x-stage variants selected by
environment variables).  Usage: xstage_ab.py OUT.npy KIND M"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1802_07844_b200 as hs  # noqa: E402
from paper_1802_07844_b200.configs import make_system  # noqa: E402

kind = sys.argv[2] if len(sys.argv) > 2 else "stokeslet"
M = int(sys.argv[3]) if len(sys.argv) > 3 else 192
name = {"stokeslet": "HL", "rotlet": "cfg4", "stresslet": "cfg3"}[kind]
s, _ = make_system(name, n=100_000)
g = hs.GridSpec(L=1.0, M=M, P=24, xi=0.26 * M)
assert g.padded_dims[0] in (480, 352), g.padded_dims
np.save(sys.argv[1], hs.fourier_space_sum(s, g).velocities)
