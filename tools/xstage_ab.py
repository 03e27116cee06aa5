"""Fourier part of a 1e5-source system on the grid of M (192 -> FFT length 480, 128 -> 352,
320 -> 750, 384 with L=2 -> 864) with the current FFT stages; saves the velocities to argv[1] (compares stage
variants selected by environment variables).  Usage: xstage_ab.py OUT.npy KIND M"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1802_07844_b200 as hs  # noqa: E402
from paper_1802_07844_b200.configs import WORKLOADS, make_system  # noqa: E402

kind = sys.argv[2] if len(sys.argv) > 2 else "stokeslet"
M = int(sys.argv[3]) if len(sys.argv) > 3 else 192
if kind == "free":
    # free space: 3 output channels (the z stage's pitch-4 interleave); M = 404 -> nz = 428, pz = 924
    s0, _ = make_system("HL", n=20_000)
    s = hs.PointSystem(kind="stokeslet", geometry="free", box_length=1.0, positions=s0.positions, f=s0.f)
    g = hs.GridSpec(L=1.0, M=M, P=24, xi=0.26 * M, geometry="free")
    assert g.padded_dims[2] == 924, g.padded_dims
    np.save(sys.argv[1], hs.fourier_space_sum(s, g).velocities)
    sys.exit(0)
if M == 384:
    assert kind == "stokeslet"
    w = WORKLOADS["cfg5"]
    s = make_system(w, n=100_000)[0].stokeslet
    g = hs.GridSpec(L=w.L, M=M, P=24, xi=w.xi)
else:
    s, _ = make_system({"stokeslet": "HL", "rotlet": "cfg4", "stresslet": "cfg3"}[kind], n=100_000)
    g = hs.GridSpec(L=1.0, M=M, P=24, xi=0.26 * M)
assert g.padded_dims[0] in (480, 352, 864, 750), g.padded_dims
np.save(sys.argv[1], hs.fourier_space_sum(s, g).velocities)
