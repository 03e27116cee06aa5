"""world_size-2 gloo tests of the target-sharded evaluation (CPU; the per-shard
evaluator is the CPU oracle, so this checks partitioning + assembly)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import hsoracle as o
    from paper_1802_07844_b200 import EwaldParams, PointSystem
    from paper_1802_07844_b200.sharding import ewald_sum_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ewald.npz"))
    s = PointSystem(kind="stresslet", geometry="half", box_length=1.0, positions=d["stresslet_pos"],
                    g=d["stresslet_g"], q=d["stresslet_q"])
    p = EwaldParams(xi=8.0, rc=0.45, M=24, P=16)
    g = o.Grid(1.0, 24, 16, 8.0)
    tabs = {t: o.precompute_greens(t, g) for t in o.table_kinds_for("stresslet", "half")}

    def evaluate(sys_, prm, _tabs, tg, ti):
        u, _, _ = o.ewald_sum("stresslet", "half", 1.0, sys_.positions, prm.xi, prm.rc, prm.M, prm.P, tabs,
                              g=sys_.g, q=sys_.q, targets=tg, target_indices=ti)
        return u

    r = ewald_sum_sharded(s, p, evaluate=evaluate)
    if rank == 0:
        np.save(out_path, r.velocities)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_cover_exactly_once():
    from paper_1802_07844_b200.sharding import shard_bounds
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            seen = np.zeros(n, int)
            for r in range(w):
                lo, hi = shard_bounds(n, w, r)
                seen[lo:hi] += 1
                assert 0 <= hi - lo <= -(-n // w)
            assert np.all(seen == 1)


def test_sharded_ewald_world2_gloo(tmp_path):
    out = str(tmp_path / "u.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    u = np.load(out)
    d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ewald.npz"))
    ref = d["stresslet_u"]   # the reference's own unsharded ewald_sum
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) < 1e-10
