"""Fourier part at the headline grid with the current x-stage; saves velocities to the path given
(used to compare x-stage variants selected by environment variables)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1802_07844_b200 as hs
from paper_1802_07844_b200.configs import make_system
kind = sys.argv[2] if len(sys.argv) > 2 else "stokeslet"
name = {"stokeslet": "HL", "rotlet": "cfg4", "stresslet": "cfg3"}[kind]
s, _ = make_system(name, n=100_000)
g = hs.GridSpec(L=1.0, M=192, P=24, xi=49.92)
np.save(sys.argv[1], hs.fourier_space_sum(s, g).velocities)
