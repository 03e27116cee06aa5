import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1802_07844_b200 as hs
d = np.load("tests/golden/ewald.npz")
s = hs.PointSystem(kind="stokeslet", geometry="half", box_length=1.0, positions=d["cfg1_pos"], f=d["cfg1_f"])
for (M, P) in ((64, 24), (64, 16), (40, 24)):
    g = hs.GridSpec(L=1.0, M=M, P=P, xi=12.0)
    uf = hs.fourier_space_sum(s, g).velocities
    z = np.where(np.all(uf == 0, axis=1))[0]
    print("M", M, "P", P, "pd", g.padded_dims, "zero rows", len(z), z[:10])
    if M == 64 and P == 24:
        ref = d["cfg1_ufourier"]
        err = np.linalg.norm(uf - ref, axis=1) / np.linalg.norm(ref, axis=1)
        print("  per-row rel err: max", err.max(), "nonzero rows max", err[~np.all(uf == 0, axis=1)].max())
        print("  zero-row positions", s.positions[z[:5]])
