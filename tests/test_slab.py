"""y-slab decomposition of one evaluation (sharding.py, csrc/plan.cu hs_slab_*).

CPU: the slab layout (every window start owned exactly once, slab heights, exchange split
sizes) and the exchange layer: DistExchange over a world-2 gloo group must move exactly
the bytes LocalExchange moves.  GPU: every rank of a W-way decomposition run in one
process (LocalExchange) reproduces the single-plan ewald_sum and the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import golden, rel_l2


def _grid(M=64, P=24, xi=12.0, L=1.0):
    from paper_1802_07844_b200.ewald import EwaldParams
    return EwaldParams(xi=xi, rc=0.1, M=M, P=P).grid(L, "half")


@pytest.mark.parametrize("M,world", [(64, 1), (64, 2), (96, 3), (192, 8), (128, 4), (384, 8)])
def test_layout_covers_planes_and_columns(M, world):
    from paper_1802_07844_b200.sharding import SlabLayout
    g = _grid(M=M)
    lay = SlabLayout(g, world)
    assert lay.y_split[0] == 0 and lay.y_split[-1] == g.dims[1]
    assert lay.kz_split[0] == 0 and lay.kz_split[-1] == g.padded_dims[2] // 2 + 1
    assert all(b > a for a, b in zip(lay.y_split, lay.y_split[1:]))
    assert all(b > a for a, b in zip(lay.kz_split, lay.kz_split[1:]))
    # ghost planes of rank r land inside rank r+1
    for r in range(world - 1):
        assert lay.y_split[r + 1] - lay.y_split[r] >= g.P - 1
    # every point's window start is owned by exactly the rank owner() names
    rng = np.random.default_rng(5)
    pts = rng.uniform(0, 1, (20000, 3))
    pts[:50, 1] = np.linspace(0, 0.999, 50)
    lo = lay.window_start_y(pts)
    own = lay.owner(pts)
    ys = np.asarray(lay.y_split)
    assert np.all(lo >= ys[own]) and np.all(lo < ys[own + 1])
    assert np.all(lo >= 0) and np.all(lo + g.P <= g.dims[1])
    # split sizes of the two all-to-alls are each other's transpose
    for r in range(world):
        for s in range(world):
            assert lay.fwd_send_splits(r)[s] == lay.fwd_recv_splits(s)[r]


def test_layout_rejects_thin_slabs():
    from paper_1802_07844_b200.errors import ParameterError
    from paper_1802_07844_b200.sharding import SlabLayout
    with pytest.raises(ParameterError):
        SlabLayout(_grid(M=64), 4)   # 65 window starts over 4 ranks < P - 1 = 23 planes


class _FakeRank:
    """Exchange buffers of one rank, filled with rank/channel-tagged values."""

    def __init__(self, lay, rank, n_in=3, n_out=2, P=24):
        self.layout, self.rank = lay, rank
        g = lay.grid
        nx, nz = int(g.dims[0]), int(g.dims[2])
        yo = lay.y_split[rank + 1] - lay.y_split[rank]
        nzl = lay.kz_split[rank + 1] - lay.kz_split[rank]
        py = int(g.padded_dims[1])
        gen = torch.Generator().manual_seed(100 + rank)
        f = lambda *s: torch.rand(*s, generator=gen, dtype=torch.float64)  # noqa: E731
        self.ghost_out, self.ghost_in = f(n_in * (P - 1) * nx * nz), torch.zeros(n_in * (P - 1) * nx * nz,
                                                                              dtype=torch.float64)
        nzh = lay.nzh
        self.send = f(n_in, 2 * yo * nx * nzh)
        self.recv = torch.zeros(n_in, 2 * py * nx * nzl, dtype=torch.float64)
        self.back = f(n_out, 2 * lay.ny * nx * nzl)
        self.recv_back = torch.zeros(n_out, 2 * yo * nx * nzh, dtype=torch.float64)
        self.halo_out = f((P - 1) * nx * nz * 6)
        self.halo_in = torch.zeros_like(self.halo_out)


def _exchange_all(xch, states):
    lay = states[0].layout
    got_g = xch.shift(states, "ghost_out", "ghost_in", +1)
    xch.all_to_all(states, "send", "recv", lay.fwd_send_splits, lay.fwd_recv_splits)
    xch.all_to_all(states, "back", "recv_back", lay.fwd_recv_splits, lay.fwd_send_splits)
    got_h = xch.shift(states, "halo_out", "halo_in", -1)
    return got_g, got_h


def _gloo_worker(rank, world, port, out_dir):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1802_07844_b200.sharding import DistExchange, LocalExchange, SlabLayout
    from paper_1802_07844_b200.ewald import EwaldParams
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = EwaldParams(xi=12.0, rc=0.1, M=40, P=8).grid(1.0, "half")
    lay = SlabLayout(g, world)
    mine = _FakeRank(lay, rank, P=8)
    got = _exchange_all(DistExchange(), [mine])
    # every process rebuilds all ranks locally (same seeds) and exchanges by copies
    allr = [_FakeRank(lay, r, P=8) for r in range(world)]
    got_l = _exchange_all(LocalExchange(), allr)
    ref = allr[rank]
    ok = all(torch.equal(getattr(mine, a), getattr(ref, a)) for a in ("ghost_in", "recv", "recv_back", "halo_in"))
    ok = ok and (rank in got[0]) == (rank in got_l[0]) and (rank in got[1]) == (rank in got_l[1])
    # per-channel asynchronous all-to-alls (the pipelined path of run_slab_pipeline)
    mine2 = _FakeRank(lay, rank, P=8)
    xch = DistExchange()
    for send_attr, recv_attr, ss, rs in (("send", "recv", lay.fwd_send_splits, lay.fwd_recv_splits),
                                         ("back", "recv_back", lay.fwd_recv_splits, lay.fwd_send_splits)):
        works = [xch.all_to_all([mine2], send_attr, recv_attr, ss, rs, channels=[c], async_op=True)
                 for c in range(getattr(mine2, send_attr).shape[0])]
        for w in works:
            xch.wait(w)
    ok = ok and torch.equal(mine2.recv, ref.recv) and torch.equal(mine2.recv_back, ref.recv_back)
    # the all-to-all really transposed: rank 1's first recv block came from rank 0
    np.save(os.path.join(out_dir, f"ok{rank}.npy"), np.array([ok]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_dist_exchange_matches_local_gloo(tmp_path, world):
    mp.spawn(_gloo_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert bool(np.load(tmp_path / f"ok{r}.npy")[0]), f"rank {r} exchange mismatch"


def test_local_exchange_transposes_blocks():
    """Block s of rank r's recv is rank s's send block r (per channel), by value."""
    from paper_1802_07844_b200.sharding import LocalExchange, SlabLayout
    from paper_1802_07844_b200.ewald import EwaldParams
    lay = SlabLayout(EwaldParams(xi=12.0, rc=0.1, M=40, P=8).grid(1.0, "half"), 3)
    st = [_FakeRank(lay, r, P=8) for r in range(3)]
    _exchange_all(LocalExchange(), st)
    for r in range(3):
        for c in range(st[r].recv.shape[0]):
            rb = st[r].recv[c, :sum(lay.fwd_recv_splits(r))].split(lay.fwd_recv_splits(r))
            for s in range(3):
                sb = st[s].send[c, :sum(lay.fwd_send_splits(s))].split(lay.fwd_send_splits(s))
                assert torch.equal(rb[s], sb[r])
    assert torch.equal(st[1].ghost_in, st[0].ghost_out) and torch.equal(st[0].halo_in, st[1].halo_out)
    assert not st[0].ghost_in.any() and not st[2].halo_in.any()


# ---------------------------------------------------------------- GPU
KINDS = ("stokeslet", "stresslet", "rotlet")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("world", [1, 2, 3])
def test_slab_local_matches_single_plan(gpu, kind, world):
    from paper_1802_07844_b200.configs import make_system
    from paper_1802_07844_b200.sharding import ewald_sum_slab_local
    name = {"stokeslet": "cfg2", "stresslet": "cfg3", "rotlet": "cfg4"}[kind]
    s, _ = make_system(name, n=20_000)
    p = gpu.EwaldParams(xi=20.8, rc=0.17, M=96, P=24)
    ref = gpu.ewald_sum(s, p)
    r = ewald_sum_slab_local(s, p, world)
    assert sum(r.meta["targets_per_rank"]) == s.n
    assert rel_l2(r.parts["real"], ref.parts["real"]) < 1e-14
    assert rel_l2(r.parts["fourier"], ref.parts["fourier"]) < 1e-12
    assert rel_l2(r.velocities, ref.velocities) < 1e-12


@pytest.mark.gpu
def test_slab_local_cfg1_vs_reference_golden(gpu):
    """BASELINE configs[0] through a 2-way slab decomposition vs the reference's own ewald_sum."""
    from paper_1802_07844_b200.sharding import ewald_sum_slab_local
    d = golden("ewald")
    s = gpu.PointSystem(kind="stokeslet", geometry="half", box_length=1.0, positions=d["cfg1_pos"], f=d["cfg1_f"])
    p = gpu.EwaldParams(xi=12.0, rc=0.35, M=64, P=24)
    r = ewald_sum_slab_local(s, p, 2)
    assert rel_l2(r.velocities, d["cfg1_u"]) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_slab_local_separate_targets(gpu, world):
    """Mixed layout: separate targets (no self term) incl. wall and top points, tables from the host."""
    from paper_1802_07844_b200.configs import make_system
    from paper_1802_07844_b200.sharding import ewald_sum_slab_local
    s, _ = make_system("cfg3", n=30_000)
    p = gpu.EwaldParams(xi=33.28, rc=0.12, M=128, P=24)
    rng = np.random.default_rng(9)
    tg = np.vstack([rng.uniform(0, 1, (5000, 3)), [[0.5, 0.0, 0.0], [0.0, 0.999, 1.0 - 1e-9]]])
    ref = gpu.ewald_sum(s, p, targets=tg)
    r = ewald_sum_slab_local(s, p, world, targets=tg)
    assert rel_l2(r.velocities, ref.velocities) < 1e-12


@pytest.mark.gpu
def test_slab_local_headline_grid_world8(gpu):
    """The headline grid (M=192) split 8 ways, at 2e5 points (every stage and exchange at HL shapes)."""
    from paper_1802_07844_b200.configs import make_system
    from paper_1802_07844_b200.sharding import ewald_sum_slab_local
    s, _ = make_system("HL", n=200_000)
    p = gpu.EwaldParams(xi=49.92, rc=0.101, M=192, P=24)
    ref = gpu.ewald_sum(s, p)
    r = ewald_sum_slab_local(s, p, 8)
    assert rel_l2(r.velocities, ref.velocities) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_slab_local_free_space(gpu, kind):
    """Free-space geometry (no images, no wall channels, the non-mirrored spread) through a
    3-way slab decomposition == the single plan."""
    from paper_1802_07844_b200.sharding import ewald_sum_slab_local
    s = gpu.generate_system(6000, 1.0, kind, "free", seed=21)
    p = gpu.EwaldParams(xi=18.0, rc=0.2, M=72, P=24)
    ref = gpu.ewald_sum(s, p)
    r = ewald_sum_slab_local(s, p, 3)
    assert rel_l2(r.velocities, ref.velocities) < 1e-12


@pytest.mark.gpu
def test_slab_local_wall_clustered_rotlet(gpu):
    """cfg4's wall-clustered rotlet (sources within a few grid cells of the wall, so the
    mirrored spread's source and image windows overlap) through a 2-way slab decomposition:
    == the single plan, and close to the direct half-space sum."""
    from paper_1802_07844_b200.configs import make_system
    from paper_1802_07844_b200.sharding import ewald_sum_slab_local
    s, _ = make_system("cfg4", n=8000)
    p = gpu.EwaldParams(xi=20.8, rc=0.17, M=96, P=24)
    ref = gpu.ewald_sum(s, p)
    r = ewald_sum_slab_local(s, p, 2)
    assert rel_l2(r.velocities, ref.velocities) < 1e-12
    d = gpu.direct_sum_half(s, targets=s.positions[:300], target_indices=np.arange(300)).velocities
    assert rel_l2(r.velocities[:300], d) < 1e-5


@pytest.mark.gpu
def test_slab_pipelined_equals_unpipelined(gpu):
    """Per-channel pipelined stages (the default) and the whole-stage calls give identical bits."""
    import torch as T
    from paper_1802_07844_b200.configs import make_system
    from paper_1802_07844_b200.sharding import (LocalExchange, SlabLayout, SlabRank, _partition_targets,
                                                _rank_inputs, run_slab_pipeline)
    s, _ = make_system("cfg3", n=12000)
    p = gpu.EwaldParams(xi=20.8, rc=0.17, M=96, P=24)
    grid = p.grid(s.box_length, s.geometry)
    lay = SlabLayout(grid, 2)
    tg, ti, rows = _partition_targets(s, lay, None, None)
    dev = T.device("cuda", 0)
    states = [SlabRank(s, p, lay, r, len(rows[r]), device=0) for r in range(2)]
    for st in states:
        st.build_tables()
    inputs = {r: _rank_inputs(s, tg, ti, rows, r, dev) for r in range(2)}
    run_slab_pipeline(states, LocalExchange(), inputs, overlap=False)
    a = [st.out[0, :len(rows[st.rank])].clone() for st in states]
    run_slab_pipeline(states, LocalExchange(), inputs, overlap=True)
    b = [st.out[0, :len(rows[st.rank])].clone() for st in states]
    assert all(T.equal(x, y) for x, y in zip(a, b))


def _gpu_slab_worker(rank, world, port, out_dir):
    """One rank of a real multi-process slab evaluation: every process drives the same GPU,
    the exchanges go through gloo with host staging (NCCL needs one GPU per rank)."""
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1802_07844_b200 import EwaldParams
    from paper_1802_07844_b200.configs import make_system
    from paper_1802_07844_b200.sharding import ewald_sum_slab
    s, _ = make_system("cfg3", n=20_000)
    r = ewald_sum_slab(s, EwaldParams(xi=20.8, rc=0.17, M=96, P=24), device=0)
    np.save(os.path.join(out_dir, f"u{rank}.npy"), r.velocities)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_slab_multiprocess_one_gpu(gpu, tmp_path, world):
    """ewald_sum_slab in `world` separate processes (DistExchange: ghost/halo P2P, per-channel
    all-to-all with uneven splits, result all-gather) == the single-plan evaluation, on every rank."""
    from paper_1802_07844_b200.configs import make_system
    mp.spawn(_gpu_slab_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    s, _ = make_system("cfg3", n=20_000)
    ref = gpu.ewald_sum(s, gpu.EwaldParams(xi=20.8, rc=0.17, M=96, P=24)).velocities
    for r in range(world):
        assert rel_l2(np.load(tmp_path / f"u{r}.npy"), ref) < 1e-12


@pytest.mark.gpu
def test_headline_full_size_vs_direct_and_slab8(gpu):
    """The metric's configuration at full size (N = 1e6, M = 192): the single plan against the
    exact O(N) direct half-space sum at 400 targets (the Ewald truncation error at these
    parameters is ~2e-11), and the 8-way y-slab decomposition against the single plan."""
    from paper_1802_07844_b200.configs import WORKLOADS, make_system
    from paper_1802_07844_b200.sharding import ewald_sum_slab_local
    w = WORKLOADS["HL"]
    s, _ = make_system(w)
    p = gpu.EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P)
    u = gpu.ewald_sum(s, p).velocities
    idx = np.random.default_rng(4).choice(s.n, 400, replace=False)
    d = gpu.direct_sum_half(s, targets=s.positions[idx], target_indices=idx).velocities
    assert rel_l2(u[idx], d) < 1e-10   # measured 2.1e-11 (the method's truncation error here)
    r = ewald_sum_slab_local(s, p, 8)
    assert rel_l2(r.velocities, u) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
def test_slab_local_mixed(gpu, world):
    """BASELINE configs[4]'s mixed stokeslet + stresslet system (separate targets) through the
    y-slab decomposition (all 19 source channels per rank, both x-stage passes on each kz
    share) == the single mixed plan."""
    from paper_1802_07844_b200.configs import make_system
    from paper_1802_07844_b200.ewald import ewald_sum_mixed
    from paper_1802_07844_b200.sharding import ewald_sum_slab_local
    s, tg = make_system("cfg5", n=20_000)
    p = gpu.EwaldParams(xi=20.8, rc=0.17, M=80, P=24)
    ref = ewald_sum_mixed(s, p, targets=tg[:6000])
    r = ewald_sum_slab_local(s, p, world, targets=tg[:6000])
    # round-off: the slab ranks add their ghost planes in a different order (measured 1.6e-12 at
    # W = 2, 3; the stresslet's near-field dominates the mixed velocities)
    assert rel_l2(r.velocities, ref.velocities) < 5e-12
