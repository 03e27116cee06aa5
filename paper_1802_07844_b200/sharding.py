"""Multi-process (one process per GPU) evaluation of ONE system, sharded by targets.

Rank r of W evaluates the targets [lo_r, hi_r) of the caller's target list
(`shard_bounds`): its real-space pair sums and Fourier gathers touch only its own
targets, while the spreading + FFT pipeline is replicated (every rank holds all
sources; the y/z-slab decomposition with NCCL transposes is the next step, see
DESIGN.md section 6).  Slices are assembled with one `all_gather` so every rank
returns the full (n_targets, 3) result, identical to the single-process one
(each target's sum is computed by exactly one rank, in the same order).

`torch.distributed` provides the plumbing: NCCL on B200 (CUDA tensors), gloo for
the CPU tests of this module (tests/test_sharding_gloo.py).
"""

from __future__ import annotations

import numpy as np

from .system import VelocityResult


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of n items for `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("invalid (world, rank)")
    base, extra = divmod(int(n), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _all_gather_rows(local: np.ndarray, n_total: int, world: int, group=None, device=None) -> np.ndarray:
    import torch
    import torch.distributed as dist
    width = local.shape[1]
    maxrows = -(-n_total // world)  # ceil
    buf = torch.zeros((maxrows, width), dtype=torch.float64, device=device)
    if local.shape[0]:
        buf[: local.shape[0]] = torch.as_tensor(local, dtype=torch.float64, device=device)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    rows = []
    for r in range(world):
        lo, hi = shard_bounds(n_total, world, r)
        rows.append(outs[r][: hi - lo].cpu().numpy())
    return np.concatenate(rows, axis=0)


def ewald_sum_sharded(system, params, tables=None, group=None, device=None, evaluate=None) -> VelocityResult:
    """ewald.ewald_sum for targets = sources (target_indices = arange(n)), sharded over the
    ranks of `group`.  `evaluate(system, params, tables, targets, target_indices)` defaults
    to the GPU `ewald_sum`; tests inject the CPU oracle to exercise the assembly on gloo."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_bounds(system.n, world, rank)
    idx = np.arange(lo, hi)
    if evaluate is None:
        from .ewald import ewald_sum

        def evaluate(sys_, p, tabs, tg, ti):
            return ewald_sum(sys_, p, tables=tabs, targets=tg, target_indices=ti).velocities
    local = np.asarray(evaluate(system, params, tables, system.positions[lo:hi], idx), dtype=np.float64)
    u = _all_gather_rows(local.reshape(-1, 3), system.n, world, group=group, device=device)
    return VelocityResult(velocities=u, meta={"kind": system.kind, "geometry": system.geometry,
                                              "shard": (rank, world, lo, hi)})


# ---------------------------------------------------------------------------
# y-slab decomposition of ONE evaluation
#
# Rank r owns grid planes y in [y0_r, y1_r) and half-spectrum columns kz in
# [kz0_r, kz1_r).  Its device plan (hs_plan_create_slab) holds every source (the
# real-space neighbourhoods and images are global) and the targets whose gather
# window starts in its slab.  One evaluation = five C stages and four exchanges:
#
#   begin     real space of the rank's targets; spread of the sources whose y window
#             starts in the slab; ghost planes [y1, y1+P-1)         --ghost-->  r+1
#   forward   ghost added; z transform; kz blocks per destination   --all-to-all (per channel)-->
#   kspace    y transform, fused x transform + k-space scaling, inverse y
#                                                                    --all-to-all (per channel)-->
#   backward  inverse z; output planes [y0, y0+P-1)                 --halo-->   r-1
#   finish    halo placed; gather; u = real + Fourier
#
# The slabs are along y (not z as SURVEY 8e sketches) because the grids are stored
# [y][x][z] with z contiguous: a y slab is one contiguous block, the z transform
# stays local, and the y/x stages run unchanged on their kz share.  The wall
# clusters sources in z (cfg4), so y slabs also balance the spreading work.
#
# Exchanges go through an `Exchange`: DistExchange (torch.distributed: NCCL on
# B200, gloo in the CPU tests) or LocalExchange (all ranks in one process,
# copies; the single-GPU test path).  The same driver runs both.

def split_range(n: int, world: int) -> list[int]:
    """Boundaries b[0..world] of a balanced split of range(n)."""
    return [shard_bounds(n, world, r)[0] for r in range(world)] + [int(n)]


class SlabLayout:
    """y planes and kz columns of every rank for one grid."""

    def __init__(self, grid, world: int):
        from ._lib import MAX_SLAB_RANKS
        from .errors import ParameterError
        if not (1 <= world <= MAX_SLAB_RANKS):
            raise ParameterError(f"slab decomposition supports 1..{MAX_SLAB_RANKS} ranks")
        self.world = int(world)
        self.grid = grid
        self.ny = int(grid.dims[1])
        self.nzh = int(grid.padded_dims[2]) // 2 + 1
        P = int(grid.P)
        # window starts lie in [0, ny - P]: split that range evenly (points, hence spreading,
        # gathering and pair work, balance with it); the last rank also owns the top P - 1 planes
        self.y_split = split_range(max(self.ny - P + 1, world), world)
        self.y_split[-1] = self.ny
        self.kz_split = split_range(self.nzh, world)
        for r in range(world - 1):
            if self.y_split[r + 1] - self.y_split[r] < P - 1:
                raise ParameterError(f"{world} y slabs of {self.ny} planes are thinner than P - 1 = {P - 1}")
        if min(self.kz_split[r + 1] - self.kz_split[r] for r in range(world)) < 1:
            raise ParameterError("more ranks than kz columns")

    def slab(self, rank: int):
        from ._lib import HsSlab
        s = HsSlab()
        s.rank, s.world = rank, self.world
        s.y0, s.y1 = self.y_split[rank], self.y_split[rank + 1]
        s.kz0, s.kz1 = self.kz_split[rank], self.kz_split[rank + 1]
        for i, v in enumerate(self.kz_split):
            s.kz_split[i] = v
        for i, v in enumerate(self.y_split):
            s.y_split[i] = v
        return s

    def window_start_y(self, points: np.ndarray) -> np.ndarray:
        """Global y window start of each point: floor((y - origin)/h) - P/2 + 1 (_gridding.py:24-25),
        the same IEEE operations as the device (common.cuh window_lo)."""
        g = self.grid
        y = np.asarray(points, dtype=np.float64)[:, 1]
        return np.floor((y - float(g.origin[1])) / float(g.h)).astype(np.int64) - int(g.P) // 2 + 1

    def owner(self, points: np.ndarray) -> np.ndarray:
        """Rank whose slab holds each point's gather window start."""
        lo = self.window_start_y(points)
        return np.clip(np.searchsorted(np.asarray(self.y_split), lo, side="right") - 1, 0, self.world - 1)

    # exchange split sizes, in doubles (complex counts 2), per channel
    def fwd_send_splits(self, rank: int) -> list[int]:
        yo = self.y_split[rank + 1] - self.y_split[rank]
        nx = int(self.grid.dims[0])
        return [2 * yo * nx * (self.kz_split[s + 1] - self.kz_split[s]) for s in range(self.world)]

    def fwd_recv_splits(self, rank: int) -> list[int]:
        nzl = self.kz_split[rank + 1] - self.kz_split[rank]
        nx = int(self.grid.dims[0])
        return [2 * (self.y_split[s + 1] - self.y_split[s]) * nx * nzl for s in range(self.world)]


class SlabRank:
    """One rank's device plan and its exchange buffers (torch CUDA tensors)."""

    def __init__(self, system, params, layout: SlabLayout, rank: int, n_targets: int, device=None):
        import torch
        from ._plan import Evaluator
        self.layout, self.rank = layout, int(rank)
        self.system = system
        grid = layout.grid
        dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
        self.device = dev
        self.ev = Evaluator(system.kind, system.geometry, system.box_length, params.xi, params.rc, grid, system.n,
                            n_targets, False, device=dev.index, slab=layout.slab(rank))
        self.lib, self.handle = self.ev.lib, self.ev.handle
        from . import _lib
        import ctypes as C
        sz = (C.c_int64 * 8)()
        _lib.check(self.lib.hs_slab_sizes(self.handle, sz))
        self.sizes = list(sz)
        n_in, n_out = self.sizes[5], self.sizes[6]
        f64 = dict(dtype=torch.float64, device=dev)
        self.ghost_out = torch.empty(self.sizes[0], **f64)
        self.ghost_in = torch.zeros(self.sizes[0], **f64)
        self.send = torch.empty((n_in, self.sizes[1]), **f64)
        self.recv = torch.zeros((n_in, self.sizes[2]), **f64)    # rows >= ny stay zero
        self.back = torch.empty((n_out, self.sizes[3]), **f64)
        self.recv_back = torch.empty((n_out, self.sizes[1]), **f64)
        self.halo_out = torch.empty(self.sizes[4], **f64)
        self.halo_in = torch.empty(self.sizes[4], **f64)
        self.n_in, self.n_out = n_in, n_out
        self.out = torch.empty((3, max(n_targets, 1), 3), **f64)
        self._inputs = None

    def _vp(self, t):
        import ctypes as C
        return C.c_void_p(t.data_ptr()) if t is not None else None

    def build_tables(self):
        self.ev.build_tables()

    def set_tables(self, tables):
        self.ev.set_tables(tables)

    def begin(self, positions, sa, sb, targets, tcols):
        from . import _lib
        self.ev.ctx.bind_torch_stream()
        self._inputs = (positions, sa, sb, targets, tcols)   # must outlive the stages
        _lib.check(self.lib.hs_slab_begin(self.handle, self._vp(positions), self._vp(sa), self._vp(sb),
                                          self._vp(targets), self._vp(tcols), _lib.HS_MEM_DEVICE,
                                          self._vp(self.ghost_out)))

    def forward(self, have_ghost: bool):
        from . import _lib
        _lib.check(self.lib.hs_slab_forward(self.handle, self._vp(self.ghost_in) if have_ghost else None,
                                            self._vp(self.send)))

    def kspace(self):
        from . import _lib
        _lib.check(self.lib.hs_slab_kspace(self.handle, self._vp(self.recv), self._vp(self.back)))

    def backward(self):
        from . import _lib
        _lib.check(self.lib.hs_slab_backward(self.handle, self._vp(self.recv_back), self._vp(self.halo_out)))

    # channel-range forms (pipelined exchanges: run_slab_pipeline(..., overlap=True))
    def forward_ch(self, have_ghost: bool, c: int):
        from . import _lib
        _lib.check(self.lib.hs_slab_forward_range(self.handle, self._vp(self.ghost_in) if have_ghost else None,
                                                  self._vp(self.send), c, c + 1))

    def kspace_in(self, c: int):
        from . import _lib
        _lib.check(self.lib.hs_slab_kspace_part(self.handle, 0, self._vp(self.recv), self._vp(self.back), c, c + 1))

    def kspace_x(self):
        from . import _lib
        _lib.check(self.lib.hs_slab_kspace_part(self.handle, 1, self._vp(self.recv), self._vp(self.back), 0, 0))

    def kspace_out(self, o: int):
        from . import _lib
        _lib.check(self.lib.hs_slab_kspace_part(self.handle, 2, self._vp(self.recv), self._vp(self.back), o, o + 1))

    def backward_ch(self, o: int):
        from . import _lib
        _lib.check(self.lib.hs_slab_backward_range(self.handle, self._vp(self.recv_back), self._vp(self.halo_out),
                                                   o, o + 1))

    def finish(self, have_halo: bool):
        import ctypes as C
        from . import _lib
        from ._plan import TIME_KEYS
        times = (C.c_double * 16)()
        u, ur, uf = self.out[0], self.out[1], self.out[2]
        _lib.check(self.lib.hs_slab_finish(self.handle, self._vp(self.halo_in) if have_halo else None,
                                           self._vp(u), self._vp(ur), self._vp(uf), _lib.HS_MEM_DEVICE, times))
        self._inputs = None
        return dict(zip(TIME_KEYS, list(times)))


class LocalExchange:
    """All ranks in this process (one device): the collectives become copies."""

    def shift(self, states, src_attr, dst_attr, step):
        """Rank r's `src_attr` buffer lands in rank r+step's `dst_attr`; returns the ranks that received."""
        got = set()
        for st in states:
            d = st.rank + step
            if 0 <= d < len(states):
                getattr(states[d], dst_attr).copy_(getattr(st, src_attr))
                got.add(d)
        return got

    def all_to_all(self, states, send_attr, recv_attr, send_splits, recv_splits, channels=None):
        n_ch = getattr(states[0], send_attr).shape[0]
        for c in (range(n_ch) if channels is None else channels):
            chunks = [getattr(st, send_attr)[c, :sum(send_splits(st.rank))].split(send_splits(st.rank))
                      for st in states]
            for st in states:
                dst = getattr(st, recv_attr)[c, :sum(recv_splits(st.rank))].split(recv_splits(st.rank))
                for s in range(len(states)):
                    dst[s].copy_(chunks[s][st.rank])
        return None

    def wait(self, handle):
        pass


class DistExchange:
    """One rank per process; torch.distributed collectives on the process group.

    staged: the group's backend cannot move device tensors (gloo): buffers go through host
    copies around each collective.  Defaults to True for a gloo group and device tensors --
    the multi-process check of the whole pipeline on one GPU (tests/test_slab.py); NCCL
    moves the device buffers directly."""

    def __init__(self, group=None, staged=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.staged = (dist.get_backend(group) == "gloo") if staged is None else bool(staged)

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def _host(self, t):
        return t.cpu() if self.staged and t.is_cuda else t

    def shift(self, states, src_attr, dst_attr, step):
        (st,) = states
        d, s = st.rank + step, st.rank - step
        src, dst = getattr(st, src_attr), getattr(st, dst_attr)
        hsrc, hdst = self._host(src), self._host(dst)
        ops = []
        if 0 <= d < self.world:
            ops.append(self.dist.P2POp(self.dist.isend, hsrc, self._peer(d), self.group))
        if 0 <= s < self.world:
            ops.append(self.dist.P2POp(self.dist.irecv, hdst, self._peer(s), self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        if hdst is not dst and 0 <= s < self.world:
            dst.copy_(hdst)
        return {st.rank} if 0 <= s < self.world else set()

    def all_to_all(self, states, send_attr, recv_attr, send_splits, recv_splits, channels=None, async_op=False):
        (st,) = states
        ss, rs = send_splits(st.rank), recv_splits(st.rank)
        src, dst = getattr(st, send_attr), getattr(st, recv_attr)
        works = []
        for c in (range(src.shape[0]) if channels is None else channels):
            if self.staged and src.is_cuda:   # host round trip, synchronous
                hd = dst[c, :sum(rs)].cpu()
                self.dist.all_to_all_single(hd, src[c, :sum(ss)].cpu(), rs, ss, group=self.group)
                dst[c, :sum(rs)].copy_(hd)
                continue
            works.append(self.dist.all_to_all_single(dst[c, :sum(rs)], src[c, :sum(ss)], rs, ss, group=self.group,
                                                     async_op=async_op))
        return works if async_op else None

    def wait(self, handle):
        # NCCL: orders the current stream after the collective (no host block); gloo: blocks
        for w in handle or ():
            w.wait()


def run_slab_pipeline(states, xch, inputs, overlap=True):
    """One sharded evaluation over the ranks in `states` (all ranks, or this process's one).

    inputs[rank] = (positions, sa, sb, targets, tcols) device tensors of that rank.
    overlap: per-channel pipelining -- the all-to-all of channel c is issued asynchronously
    (DistExchange: on the collective's stream) right after channel c is transformed, so it
    overlaps the z / y transforms of the next channels.  Returns {rank: times}."""
    lay = states[0].layout
    for st in states:
        st.begin(*inputs[st.rank])
    got = xch.shift(states, "ghost_out", "ghost_in", +1)
    if not overlap:
        for st in states:
            st.forward(st.rank in got)
        xch.all_to_all(states, "send", "recv", lay.fwd_send_splits, lay.fwd_recv_splits)
        for st in states:
            st.kspace()
        xch.all_to_all(states, "back", "recv_back", lay.fwd_recv_splits, lay.fwd_send_splits)
        for st in states:
            st.backward()
    else:
        n_in, n_out = states[0].n_in, states[0].n_out
        kw = {"async_op": True} if isinstance(xch, DistExchange) else {}
        pend = []
        for c in range(n_in):
            for st in states:
                st.forward_ch(st.rank in got, c)
            pend.append(xch.all_to_all(states, "send", "recv", lay.fwd_send_splits, lay.fwd_recv_splits,
                                       channels=[c], **kw))
        for c in range(n_in):
            xch.wait(pend[c])
            for st in states:
                st.kspace_in(c)
        for st in states:
            st.kspace_x()
        pend = []
        for o in range(n_out):
            for st in states:
                st.kspace_out(o)
            pend.append(xch.all_to_all(states, "back", "recv_back", lay.fwd_recv_splits, lay.fwd_send_splits,
                                       channels=[o], **kw))
        for o in range(n_out):
            xch.wait(pend[o])
            for st in states:
                st.backward_ch(o)
    got = xch.shift(states, "halo_out", "halo_in", -1)
    return {st.rank: st.finish(st.rank in got) for st in states}


def _partition_targets(system, layout: SlabLayout, targets, target_indices):
    """(positions, target_indices) of every rank's targets and the original row of each."""
    if targets is None:
        tg = np.asarray(system.positions, dtype=np.float64)
        ti = np.arange(system.n, dtype=np.int64)
    else:
        tg = np.atleast_2d(np.asarray(targets, dtype=np.float64))
        ti = (np.full(tg.shape[0], -1, dtype=np.int64) if target_indices is None
              else np.asarray(target_indices, dtype=np.int64))
    own = layout.owner(tg)
    rows = [np.nonzero(own == r)[0] for r in range(layout.world)]
    return tg, ti, rows


def _rank_inputs(system, tg, ti, rows, rank, dev):
    import torch
    from .ewald import _strengths
    sa, sb = _strengths(system)
    t = lambda a: None if a is None else torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)  # noqa: E731
    r = rows[rank]
    return (t(system.positions), t(sa), t(sb), t(tg[r].reshape(-1, 3)),
            torch.as_tensor(np.ascontiguousarray(ti[r]), device=dev))


def _prepare_rank_tables(st, system, grid, tables):
    from .ewald_fourier import check_tables, table_kinds_for
    if tables is None:
        st.build_tables()
    else:
        check_tables(system, grid, tables)
        st.set_tables({k: tables[k] for k in table_kinds_for(system.kind, grid.geometry)})


def ewald_sum_slab_local(system, params, world: int, tables=None, targets=None, target_indices=None,
                         device=None) -> VelocityResult:
    """ewald.ewald_sum through the y-slab decomposition with all `world` ranks in this process
    on one device (LocalExchange).  Exercises every stage and exchange layout of the
    multi-GPU path on a single GPU; the result must equal the single-plan evaluation."""
    import torch
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    grid = params.grid(system.box_length, system.geometry)
    lay = SlabLayout(grid, world)
    tg, ti, rows = _partition_targets(system, lay, targets, target_indices)
    states = [SlabRank(system, params, lay, r, len(rows[r]), device=dev.index) for r in range(world)]
    for st in states:
        _prepare_rank_tables(st, system, grid, tables)
    inputs = {r: _rank_inputs(system, tg, ti, rows, r, dev) for r in range(world)}
    times = run_slab_pipeline(states, LocalExchange(), inputs)
    u = np.zeros((tg.shape[0], 3))
    ur, uf = np.zeros_like(u), np.zeros_like(u)
    for st in states:
        k = len(rows[st.rank])
        u[rows[st.rank]] = st.out[0, :k].cpu().numpy()
        ur[rows[st.rank]] = st.out[1, :k].cpu().numpy()
        uf[rows[st.rank]] = st.out[2, :k].cpu().numpy()
    return VelocityResult(velocities=u, parts={"real": ur, "fourier": uf},
                          meta={"kind": system.kind, "geometry": system.geometry, "slab_world": world,
                                "targets_per_rank": [len(r) for r in rows], "times_ms": times})


_slab_cache: dict = {}


def slab_rank(system, params, group=None, targets=None, target_indices=None, device=None):
    """This process's SlabRank (cached per configuration), its layout and target partition."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    grid = params.grid(system.box_length, system.geometry)
    lay = SlabLayout(grid, world)
    tg, ti, rows = _partition_targets(system, lay, targets, target_indices)
    key = (system.kind, system.geometry, float(system.box_length), params.xi, params.rc, params.M, params.P,
           system.n, len(rows[rank]), world, rank, device)
    st = _slab_cache.get(key)
    if st is None:
        _slab_cache.clear()
        st = SlabRank(system, params, lay, rank, len(rows[rank]), device=device)
        _slab_cache[key] = st
    return st, lay, tg, ti, rows


def ewald_sum_slab(system, params, tables=None, group=None, targets=None, target_indices=None,
                   device=None) -> VelocityResult:
    """ewald.ewald_sum of ONE system over the ranks of `group`, y-slab decomposed (one process per
    GPU, NCCL).  Every rank passes the same system and returns the full (n_targets, 3) result
    (its own rows computed locally, the others all-gathered)."""
    import torch
    import torch.distributed as dist
    st, lay, tg, ti, rows = slab_rank(system, params, group, targets, target_indices, device)
    grid = lay.grid
    if not st.ev.tables_ready:
        _prepare_rank_tables(st, system, grid, tables)
    inputs = {st.rank: _rank_inputs(system, tg, ti, rows, st.rank, st.device)}
    times = run_slab_pipeline([st], DistExchange(group), inputs)[st.rank]
    k = len(rows[st.rank])
    kmax = max(len(r) for r in rows)
    buf = torch.zeros((3, max(kmax, 1), 3), dtype=torch.float64, device=st.device)
    buf[:, :k] = st.out[:, :k]
    outs = [torch.empty_like(buf) for _ in range(lay.world)]
    dist.all_gather(outs, buf, group=group)
    full = np.zeros((3, tg.shape[0], 3))
    for r in range(lay.world):
        full[:, rows[r]] = outs[r][:, :len(rows[r])].cpu().numpy()
    return VelocityResult(velocities=full[0], parts={"real": full[1], "fourier": full[2]},
                          meta={"kind": system.kind, "geometry": system.geometry, "slab": (st.rank, lay.world),
                                "targets_per_rank": [len(r) for r in rows], "times_ms": times})
