"""Plan cache and evaluator around the C ABI's hs_plan (csrc/plan.cu).

An :class:`Evaluator` owns one device plan for a fixed (kind, geometry, grid,
rc, n, n_targets) configuration and evaluates it for new strengths/positions.
Inputs may be NumPy arrays (host; copied by the library on its stream) or
torch CUDA tensors (device-resident; zero copies).
"""

from __future__ import annotations

import ctypes as C
import math
import gc
import threading

import numpy as np

from . import _lib
from .errors import ResourceError, ParameterError

TIME_KEYS = ("gridding", "fft", "scale", "ifft", "gather", "real", "fourier", "prep", "total", "io",
             "k_pair", "k_spread", "k_gather", "k_scale", "pairs", "image_pairs")


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _host_f64(a, shape_cols=3):
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if arr.ndim != 2 or arr.shape[1] != shape_cols:
        raise ParameterError(f"expected (n,{shape_cols}) float64 array, got {arr.shape}")
    return arr


class Evaluator:
    """Device plan for one configuration (grid from a GridSpec-like object)."""

    def __init__(self, kind, geometry, L, xi, rc, grid, n, n_targets, targets_are_sources, device=None, slab=None):
        self.ctx = _lib.Context.get(device)
        self.lib = self.ctx.lib
        self.kind, self.geometry = kind, geometry
        self.n, self.n_targets = int(n), int(n_targets)
        self.targets_are_sources = bool(targets_are_sources)
        self.grid = grid
        p = _lib.HsParams()
        p.kind = _lib.KIND_ID[kind]
        p.geometry = _lib.GEOM_ID[geometry]
        p.L = float(L)
        p.xi = float(xi)
        p.rc = float(rc)
        p.M = int(grid.M)
        p.P = int(grid.P)
        p.h = float(grid.h)
        p.eta = float(grid.eta)
        p.origin = _lib.vec3([float(v) for v in grid.origin])
        p.dims = _lib.vec3([int(v) for v in grid.dims], C.c_int64)
        p.padded = _lib.vec3([int(v) for v in grid.padded_dims], C.c_int64)
        p.n = self.n
        p.n_targets = self.n_targets
        p.targets_are_sources = 1 if self.targets_are_sources else 0
        self.params = p
        self._b_cols = 6 if kind == "mixed" else 3   # mixed: sb rows are [g | q]
        h = C.c_void_p()
        if slab is None:
            _lib.check(self.lib.hs_plan_create(self.ctx.handle, C.byref(p), C.byref(h)))
        else:   # y-slab share of a sharded evaluation (sharding.py)
            _lib.check(self.lib.hs_plan_create_slab(self.ctx.handle, C.byref(p), C.byref(slab), C.byref(h)))
        self.handle = h
        self._table_ids = {}
        self.tables_ready = False

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.hs_plan_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def device_bytes(self) -> int:
        return int(self.lib.hs_plan_bytes(self.handle))

    def fft_counts(self):
        a, b = C.c_int(), C.c_int()
        _lib.check(self.lib.hs_plan_fft_counts(self.handle, C.byref(a), C.byref(b)))
        return a.value, b.value

    # ---- tables
    def build_tables(self):
        """GPU precompute_greens for every table this kind/geometry needs (ewald_fourier.py:207-244)."""
        from .ewald_fourier import _oversampling_big
        big = np.asarray(_oversampling_big(self.grid), dtype=np.int64)
        guards = np.asarray(self.grid.guards, dtype=np.int64)
        _lib.check(self.lib.hs_plan_build_tables(self.handle, _lib.i64ptr(big), float(self.grid.R),
                                                 _lib.i64ptr(guards)))
        self.tables_ready = True
        self._table_ids = {"built": True}

    def set_tables(self, tables: dict):
        """Load reference-layout GreensTable samples (host or torch CUDA)."""
        for name, tab in tables.items():
            key = (id(tab), id(getattr(tab, "samples", None)))
            if self._table_ids.get(name) == key:
                continue
            s = tab.samples
            if _is_torch(s):
                s = s.contiguous()
                _lib.check(self.lib.hs_plan_set_table(self.handle, _lib.TABLE_ID[name], C.c_void_p(s.data_ptr()),
                                                      _lib.HS_MEM_DEVICE))
            else:
                arr = np.ascontiguousarray(s, dtype=np.float64)
                _lib.check(self.lib.hs_plan_set_table(self.handle, _lib.TABLE_ID[name],
                                                      arr.ctypes.data_as(C.c_void_p), _lib.HS_MEM_HOST))
            self._table_ids[name] = key
        self.tables_ready = True

    # ---- evaluation
    def execute(self, positions, sa, sb=None, targets=None, tcols=None, what=3, out=None):
        """Run the plan.  Host (NumPy) inputs -> NumPy outputs; torch CUDA inputs -> torch outputs.

        Returns (u, u_real, u_fourier, times_ms dict)."""
        times = (C.c_double * 16)()
        if _is_torch(positions):
            return self._execute_torch(positions, sa, sb, targets, tcols, what, times, out)
        pos = _host_f64(positions)
        a = _host_f64(sa)
        b = _host_f64(sb, self._b_cols) if sb is not None else None
        nt = self.n_targets
        tg = _host_f64(targets) if targets is not None else None
        tc = np.ascontiguousarray(np.asarray(tcols, dtype=np.int64)) if tcols is not None else None
        self._check_rows(pos, a, b, tg, tc)
        if out is not None:   # caller-provided (e.g. pinned) host buffers; parts may be None
            u, ur, uf = out
        else:
            u, ur, uf = np.empty((nt, 3)), np.empty((nt, 3)), np.empty((nt, 3))
        vp = lambda x: x.ctypes.data_as(C.c_void_p) if x is not None else None  # noqa: E731
        self.ctx.bind_stream(None)
        st = self.lib.hs_plan_execute(self.handle, vp(pos), vp(a), vp(b), vp(tg), vp(tc), vp(u), vp(ur), vp(uf),
                                      _lib.HS_MEM_HOST, int(what), times)
        _lib.check(st)
        return u, ur, uf, dict(zip(TIME_KEYS, list(times)))

    def pair_audit(self, positions, sa, sb=None, targets=None, tcols=None):
        """Per-target neighbour audit of the real-space pass (hs_plan_pair_audit): uint64
        (n_targets, 3) = [accepted pairs, accepted image pairs, sum of splitmix64(id) mod 2^64]."""
        pos = _host_f64(positions)
        a = _host_f64(sa)
        b = _host_f64(sb, self._b_cols) if sb is not None else None
        tg = _host_f64(targets) if targets is not None else None
        tc = np.ascontiguousarray(np.asarray(tcols, dtype=np.int64)) if tcols is not None else None
        self._check_rows(pos, a, b, tg, tc)
        out = np.zeros((self.n_targets, 3), dtype=np.uint64)
        vp = lambda x: x.ctypes.data_as(C.c_void_p) if x is not None else None  # noqa: E731
        self.ctx.bind_stream(None)
        _lib.check(self.lib.hs_plan_pair_audit(self.handle, vp(pos), vp(a), vp(b), vp(tg), vp(tc), vp(out),
                                               _lib.HS_MEM_HOST))
        return out

    def _check_rows(self, pos, a, b, tg, tc):
        if pos.shape[0] != self.n or a.shape[0] != self.n or (b is not None and b.shape[0] != self.n):
            raise ParameterError(f"plan expects {self.n} sources")
        if self.kind != "stokeslet" and b is None:
            raise ParameterError(f"{self.kind} needs q")
        if not self.targets_are_sources:
            if tg is None or tg.shape[0] != self.n_targets:
                raise ParameterError(f"plan expects {self.n_targets} targets")
            if tc is not None and tc.shape != (self.n_targets,):
                raise ParameterError("target_indices must have one entry per target")

    def _check_torch(self, dev, **tensors):
        """Device inputs are passed to the kernels as raw pointers: dtype, layout, device and row
        count must match exactly (float64 (rows,3) / int64 (rows,), contiguous, on the plan's device)."""
        import torch
        rows = {"positions": self.n, "sa": self.n, "sb": self.n, "targets": self.n_targets,
                "tcols": self.n_targets}
        for name, t in tensors.items():
            if t is None:
                continue
            want = torch.int64 if name == "tcols" else torch.float64
            shape = (rows[name],) if name == "tcols" else (rows[name], self._b_cols if name == "sb" else 3)
            if not isinstance(t, torch.Tensor) or t.dtype != want or not t.is_cuda or t.device != dev \
                    or tuple(t.shape) != shape or not t.is_contiguous():
                raise ParameterError(f"{name}: expected a contiguous {want} CUDA tensor of shape {shape} on {dev}, "
                                     f"got {getattr(t, 'dtype', type(t))} {tuple(getattr(t, 'shape', ()))} "
                                     f"on {getattr(t, 'device', '?')}")
        if self.kind != "stokeslet" and tensors.get("sb") is None:
            raise ParameterError(f"{self.kind} needs q")
        if not self.targets_are_sources and tensors.get("targets") is None:
            raise ParameterError(f"plan expects {self.n_targets} targets")

    def _execute_torch(self, positions, sa, sb, targets, tcols, what, times, out):
        import torch
        dev = positions.device
        if self.ctx.device is not None and dev.index != self.ctx.device:
            raise ParameterError(f"inputs on {dev}, plan on cuda:{self.ctx.device}")
        self._check_torch(dev, positions=positions, sa=sa, sb=sb, targets=targets, tcols=tcols)
        nt = self.n_targets
        if out is None:
            out = torch.empty((3, nt, 3), dtype=torch.float64, device=dev)
        u, ur, uf = out[0], out[1], out[2]
        vp = lambda x: C.c_void_p(x.data_ptr()) if x is not None else None  # noqa: E731
        self.ctx.bind_torch_stream()
        st = self.lib.hs_plan_execute(self.handle, vp(positions), vp(sa), vp(sb), vp(targets), vp(tcols), vp(u),
                                      vp(ur), vp(uf), _lib.HS_MEM_DEVICE, int(what), times)
        _lib.check(st)
        return u, ur, uf, dict(zip(TIME_KEYS, list(times)))


_cache: dict = {}
_cache_lock = threading.Lock()
_CACHE_MAX = 4


def get_evaluator(kind, geometry, L, xi, rc, grid, n, n_targets, targets_are_sources) -> Evaluator:
    key = (kind, geometry, float(L), float(xi), float(rc), int(grid.M), int(grid.P), tuple(grid.padded_dims),
           int(n), int(n_targets), bool(targets_are_sources))
    with _cache_lock:
        ev = _cache.get(key)
        if ev is None:
            while len(_cache) >= _CACHE_MAX:
                _cache.pop(next(iter(_cache)))
            try:
                ev = Evaluator(kind, geometry, L, xi, rc, grid, n, n_targets, targets_are_sources)
            except ResourceError:
                # device memory held by cached plans of other shapes: release them and retry once
                _cache.clear()
                gc.collect()
                ev = Evaluator(kind, geometry, L, xi, rc, grid, n, n_targets, targets_are_sources)
            _cache[key] = ev
        return ev


def clear_cache():
    with _cache_lock:
        _cache.clear()
