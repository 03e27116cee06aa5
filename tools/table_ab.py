"""Build one Green's table on the GPU and save it (compares table-precompute variants selected by
environment variables).  Usage: table_ab.py OUT.npy KIND(harmonic|biharmonic) M"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1802_07844_b200 as hs  # noqa: E402

kind, M = sys.argv[2], int(sys.argv[3])
g = hs.GridSpec(L=1.0, M=M, P=24, xi=0.26 * M)
np.save(sys.argv[1], hs.precompute_greens(kind, g, max_bytes=None).samples)
