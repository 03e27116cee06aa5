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
