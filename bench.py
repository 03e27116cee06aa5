#!/usr/bin/env python
"""Headline benchmark: half-space stokeslet Ewald target evaluations/s at N=1e6, FP64
(BASELINE.json `metric`, workload "HL": N=1e6, xi=49.92, r_c=0.101, M=192, P=24).

One step = one full ewald_sum evaluation (real + Fourier) of the whole system,
inputs resident in HBM, Green's tables precomputed outside the timed region (as
the reference and the paper do).  `e2e` repeats the measurement through the
C ABI with pinned HOST buffers (H2D of positions+forces and D2H of velocities
inside the timed region).  `--impl reference` times the CPU restatement of the
reference (oracle/, OpenMP C + scipy.fft) on a bounded sample of the same
workload, extrapolated to the full evaluation.

Multi-GPU (torchrun), two modes:
  --mode replicas (default): every rank evaluates its own independent HL system
      (weak scaling, no data-path collective);
  --mode slab: ONE system y-slab decomposed over the ranks (sharding.py: spread
      ghost planes, per-channel NCCL all-to-all transposes of the FFT, gather halo;
      strong scaling, value = N / time of one sharded evaluation).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "half-space stokeslet Ewald target evals/sec @N=1e6 FP64"
UNIT = "target_evals/s"
FP64_PEAK_SOURCE = os.path.join(ROOT, "profiles", "r01_probe_fp64.json")


def _peaks():
    hbm, fp64, src = 6549.1, None, "fallback"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        hbm = float(json.load(open(p))["hbm_gbs"])
        src = "MEASURED_PEAKS.json"
    if os.path.exists(FP64_PEAK_SOURCE):
        d = json.load(open(FP64_PEAK_SOURCE))
        fp64 = {"dfma": d["dfma_tflops"], "dmma": d["dmma_tflops"]}
    return hbm, fp64 or {"dfma": 33.9, "dmma": 37.1}, src


# ---------------------------------------------------------------------------
# CPU baseline: oracle port (test infrastructure), bounded sample, extrapolated
def cpu_sample(wname: str, threads: int | None = None):
    """Estimate seconds for one full ewald_sum evaluation of the workload on host cores."""
    from oracle import hsoracle as o
    from paper_1802_07844_b200.configs import WORKLOADS, make_system
    import scipy.fft as sfft
    w = WORKLOADS[wname]
    threads = threads or os.cpu_count()
    o.set_threads(threads)
    s, _ = make_system(w)
    n = s.n
    pos, f = s.positions, s.f
    g = o.Grid(w.L, w.M, w.P, w.xi, "half")
    rng = np.random.default_rng(0)
    parts = {}
    t_wall = time.perf_counter()
    zz, sa, sb, sign = o.reflect(pos, "stokeslet", f=f)
    # real space: set-up (reflection, cell list of all 2N points, permutations) once; the
    # pair loop on a sample of targets, scaled
    nts = min(n, 48000)
    sub = np.sort(rng.choice(n, nts, replace=False))
    tr = {}
    o.real_space_sum("stokeslet", "half", w.L, pos, w.xi, w.rc, f=f, targets=pos[sub], target_indices=sub,
                     timings=tr)
    parts["real"] = tr["setup"] + tr["pairs"] * n / nts
    # spreading: the scatter loop on a sample of sources (3 kernel + 4 wall channels), scaled;
    # grid zeroing and the channel-first copy at full size
    frac = min(1.0, 240000 / (2 * n))
    ks = rng.choice(2 * n, int(2 * n * frac), replace=False)
    s_, v_, _ = o.phi_channels("stokeslet", pos, f=f)
    cs = rng.choice(n, int(n * frac), replace=False)
    t1, t2 = {}, {}
    o.spread(zz[ks], sa[ks], g, timings=t1)
    o.spread((pos * [1, 1, -1])[cs], np.column_stack([s_, v_])[cs], g, timings=t2)
    parts["gridding"] = (t1["loop"] + t2["loop"]) / frac + t1["copy"] + t2["copy"]
    # FFTs: one forward and one inverse on a 1/8-volume grid, scaled by N log N
    pd = g.padded_dims
    sd = tuple(p // 2 for p in pd)
    buf = np.zeros(sd)
    buf[: sd[0] // 2, : sd[1] // 2, : sd[2] // 2] = rng.normal(size=(sd[0] // 2, sd[1] // 2, sd[2] // 2))
    t0 = time.perf_counter()
    spec = sfft.fftn(buf, workers=threads)
    tf = time.perf_counter() - t0
    t0 = time.perf_counter()
    sfft.ifftn(spec, workers=threads)
    ti = time.perf_counter() - t0
    del spec, buf
    nfull, nsmall = float(np.prod(pd)), float(np.prod(sd))
    sc = nfull * math.log2(nfull) / (nsmall * math.log2(nsmall))
    parts["fft"] = 7 * tf * sc
    parts["ifft"] = 6 * ti * sc
    # k-space scaling (kernel + wall channels) on a slab of planes
    planes = 36
    shp = (planes, pd[1], pd[2])
    Ch = (rng.normal(size=(3,) + shp) + 1j * rng.normal(size=(3,) + shp))
    tab = rng.normal(size=shp)
    k1 = [2.0 * math.pi * sfft.fftfreq(p, d=g.h) for p in pd]
    out = np.empty((3,) + shp, np.complex128)
    t0 = time.perf_counter()
    o.lib().or_kspace_scale(0, o._d(Ch.view(np.float64)), o._d(tab), o._d(k1[0][:planes]), o._d(k1[1]), o._d(k1[2]),
                            planes, pd[1], pd[2], 0.1, 0.1, out.view(np.float64).ctypes.data_as(
                                o.C.POINTER(o.C.c_double)))
    kx, ky, kz = k1[0][:planes, None, None], k1[1][None, :, None], k1[2][None, None, :]
    Fc = tab * np.exp(-0.1 * (kx**2 + ky**2 + kz**2))
    phi = Fc * Ch[0]
    for j, kk in enumerate((kx, ky, kz)):
        phi = phi + 1j * kk * (Fc * Ch[j])
    parts["scale"] = (time.perf_counter() - t0) * pd[0] / planes
    del Ch, out, phi, Fc, tab
    # gather: 6 channels at a target sample
    grids = np.zeros((3,) + tuple(g.dims))
    ntg = 18000
    tg = {}
    o.gather(grids, pos[:ntg], g, timings=tg)
    parts["gather"] = 2 * (tg["copy"] + tg["loop"] * n / ntg)
    del grids
    total = sum(parts.values())
    sample_desc = (f"oracle port ({threads} threads): set-up + cell list at full size; pair loop for {nts} sampled targets; spread of "
                   f"{frac:.3%} of sources; fwd+inv FFT on a 1/8-volume grid scaled by NlogN (x7 fwd, x6 inv); "
                   f"k-space scale on {planes}/{pd[0]} planes; gather at {ntg} targets; each scaled to N={n}")
    return total, parts, sample_desc, time.perf_counter() - t_wall, threads


# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        os.unlink(self.path)
        sm = [float(r[0]) for r in rows if len(r) >= 8 and r[0].strip().replace(".", "").isdigit()]
        if not sm:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(float(r[1]) for r in rows),
                "samples": len(sm), "reasons": sorted(reasons)}


def roofline(times, work, hbm_peak, fp64_peak):
    """Per-kernel achieved vs peak.  work: algorithmic FLOP or bytes per launch."""
    ks = {}
    for name, (kind, amount, bound) in work.items():
        t = times.get(name)
        if not t or t <= 0:
            continue
        if bound == "hbm":
            ach = amount / (t * 1e-3) / 1e9
            ks[name] = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                        "ms": t, "algorithmic": amount}
        else:
            pk = fp64_peak[bound.split(":")[1]]  # "fp64:dfma" (FP64 FMA pipe) or "fp64:dmma" (FP64 tensor pipe)
            ach = amount / (t * 1e-3) / 1e12
            ks[name] = {"bound": "fp64", "pipe": bound.split(":")[1], "achieved": ach, "peak": pk,
                        "unit": "TFLOP/s", "frac": ach / pk, "ms": t, "algorithmic": amount}
    return ks


def run_reference(args, rank):
    if rank != 0:
        return
    from paper_1802_07844_b200.configs import WORKLOADS
    w = WORKLOADS[args.workload]
    for _ in range(args.warmup):
        cpu_sample(args.workload)
    vals, walls = [], []
    last = None
    for _ in range(args.steps):
        total, parts, desc, wall, thr = cpu_sample(args.workload)
        vals.append(total)
        walls.append(wall)
        last = (parts, desc, thr)
    t = float(np.mean(vals))
    value = w.n / t
    parts, desc, thr = last
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded PCG64, BASELINE.json shapes)",
            "config": {"workload": w.name, "kind": w.kind, "n": w.n, "xi": w.xi, "rc": w.rc, "M": w.M, "P": w.P},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "port", "sample": desc,
                             "phases_s": {k: round(v, 4) for k, v in parts.items()},
                             "sample_wall_s": round(float(np.mean(walls)), 2)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1802_07844_b200 import GridSpec, _lib
    from paper_1802_07844_b200._plan import Evaluator
    from paper_1802_07844_b200.configs import WORKLOADS, Workload, make_system

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    w0 = WORKLOADS[args.workload]
    w = Workload(**{**w0.__dict__, "seed": w0.seed + 7919 * rank})   # replicas: independent systems
    s, targets = make_system(w)
    grid = GridSpec(L=w.L, M=w.M, P=w.P, xi=w.xi, geometry="half")
    ev = Evaluator(w.kind, "half", w.L, w.xi, w.rc, grid, s.n, s.n if targets is None else targets.shape[0],
                   targets is None, device=local_rank)
    t0 = time.perf_counter()
    ev.build_tables()
    t_tables = time.perf_counter() - t0
    dev = torch.device("cuda", local_rank)
    pos = torch.from_numpy(s.positions).to(dev)
    f = torch.from_numpy(s.f).to(dev)
    out = torch.empty((3, s.n, 3), dtype=torch.float64, device=dev)
    for _ in range(args.warmup):
        ev.execute(pos, f, out=out)
    torch.cuda.synchronize()
    ctx = _lib.Context.get(local_rank)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.25)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step_times = []
    for _ in range(args.steps):
        _, _, _, tm = ev.execute(pos, f, out=out)
        step_times.append(tm)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launches() - l0
    clk = clocks.stop()
    # per-kernel times for the roofline: the same evaluations with the real-space and Fourier
    # pipelines serialised (what bit 2), since in the timed steps they overlap on two streams
    # and a kernel's event interval would include the other pipeline's work
    step_times = []
    for _ in range(args.steps):
        _, _, _, tm = ev.execute(pos, f, out=out, what=7)
        step_times.append(tm)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    value = world * s.n * args.steps / (ms * 1e-3)
    avg = {k: float(np.mean([t[k] for t in step_times])) for k in step_times[0]}

    # ---- e2e through the C ABI with pinned host buffers
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hp, hf = pin(s.positions), pin(s.f)
    hu = torch.empty((s.n, 3), dtype=torch.float64).pin_memory()
    hpos, hfor, hout = hp.numpy(), hf.numpy(), hu.numpy()
    ev.execute(hpos, hfor, out=(hout, None, None))   # warm
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        ev.execute(hpos, hfor, out=(hout, None, None))
    e1.record()
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_e2e = float(tt.item())
    e2e_value = world * s.n * args.steps / (ms_e2e * 1e-3)
    # parity spot-check of the e2e result against the device result
    dev_u = out[0].cpu().numpy()
    e2e_consistent = bool(np.array_equal(dev_u, hout))

    # ---- roofline (algorithmic work per launch)
    hbm_peak, fp64_peak, peak_src = _peaks()
    P3 = w.P ** 3
    n_half = grid.padded_dims[0] * grid.padded_dims[1] * (grid.padded_dims[2] // 2 + 1)
    pairs, img_pairs = avg["pairs"], avg["image_pairs"]
    work = {
        # mirrored spreading (csrc/plan.cu k_mirror_z): 3 kernel + 4 wall channels at the N
        # sources, images by reflection of the grid (10 N P^3 -> 7 N P^3 FMAs)
        "k_spread": ("flop", 2.0 * P3 * 7 * s.n, "fp64:dmma"),
        "k_gather": ("flop", 2.0 * P3 * 6 * s.n, "fp64:dfma"),
        "k_scale": ("bytes", n_half * (16 * 7 + 16 * 6 + 8 * 2), "hbm"),
        "k_pair": ("flop", 2.0 * (64 * pairs + 33 * img_pairs), "fp64:dfma"),
    }
    kern = roofline(avg, work, hbm_peak, fp64_peak)
    dom = max(kern, key=lambda k: kern[k]["ms"])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_per_launch.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(dom)
    rf = dict(kern[dom])
    rf.update({"kernel": dom, "traffic": traffic, "peak_source": (
        "MEASURED_PEAKS.json hbm_gbs" if rf["bound"] == "hbm" else
        f"measured FP64 {rf['pipe'].upper()} microbenchmark, profiles/r01_probe_fp64.json")})

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded PCG64, BASELINE.json shapes)",
            "config": {"workload": w.name, "kind": w.kind, "n": s.n, "xi": w.xi, "rc": w.rc, "M": w.M, "P": w.P,
                       "padded_dims": list(grid.padded_dims), "parallelism": f"replicas{world}",
                       "streams": "real space concurrent with the Fourier pipeline up to the gather; "
                                  "kernels/phases_ms/roofline from the same steps run serialised",
                       "l2": "not flushed: each step streams >30 GB of grids/spectra through HBM (126 MB L2)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(hp.numel() * 8 + hf.numel() * 8),
                    "d2h_bytes_per_step": int(hu.numel() * 8), "ms_per_step": ms_e2e / args.steps,
                    "matches_device_result": e2e_consistent},
            "gpu_launches": int(launches), "gpu_launches_note": "hand-written kernels only; cuFFT launches excluded",
            "roofline": rf, "kernels": kern,
            "phases_ms": {k: round(avg[k], 4) for k in ("real", "gridding", "fft", "scale", "ifft", "gather",
                                                        "total")},
            "pairs_per_step": pairs, "image_pairs_per_step": img_pairs,
            "precompute_tables_s": round(t_tables, 3), "plan_device_bytes": ev.device_bytes,
            "clocks": clk}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        total, parts, desc, wall, thr = cpu_sample(args.workload)
        line["cpu_baseline"] = {"value": s.n / total, "unit": UNIT, "cores": thr, "kind": "port", "sample": desc,
                                "phases_s": {k: round(v, 4) for k, v in parts.items()},
                                "sample_wall_s": round(wall, 2)}
    if rank == 0:
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def run_slab(args, rank, world, local_rank):
    """One system, y-slab decomposed over `world` ranks (strong scaling)."""
    import torch
    import torch.distributed as dist
    from paper_1802_07844_b200 import EwaldParams, _lib
    from paper_1802_07844_b200.configs import WORKLOADS, make_system
    from paper_1802_07844_b200.sharding import DistExchange, _rank_inputs, run_slab_pipeline, slab_rank

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo", device_id=dev,
                            rank=rank, world_size=world)
    w = WORKLOADS[args.workload]
    s, targets = make_system(w)
    p = EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P)
    st, lay, tg, ti, rows = slab_rank(s, p, targets=targets, device=local_rank)
    t0 = time.perf_counter()
    st.build_tables()
    t_tables = time.perf_counter() - t0
    inputs = {rank: _rank_inputs(s, tg, ti, rows, rank, dev)}
    xch = DistExchange()
    for _ in range(args.warmup):
        run_slab_pipeline([st], xch, inputs)
    ctx = _lib.Context.get(local_rank)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.25)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step_times = []
    for _ in range(args.steps):
        step_times.append(run_slab_pipeline([st], xch, inputs)[rank])
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    launches = ctx.launches() - l0
    clk = clocks.stop()
    tt = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    n_t = tg.shape[0]
    value = n_t * args.steps / (ms * 1e-3)
    # e2e: this rank's inputs copied from pinned host memory and its rows read back, every step
    pin = [None if a is None else a.cpu().pin_memory() for a in inputs[rank]]
    hu = torch.empty((max(len(rows[rank]), 1), 3), dtype=torch.float64).pin_memory()
    bi = sum(a.numel() * a.element_size() for a in pin if a is not None)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        dins = {rank: tuple(None if a is None else a.to(dev, non_blocking=True) for a in pin)}
        run_slab_pipeline([st], xch, dins)
        hu.copy_(st.out[0, :hu.shape[0]], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    tt = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_e2e = float(tt.item())
    avg = {k: float(np.mean([t[k] for t in step_times])) for k in step_times[0]}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded PCG64, BASELINE.json shapes)",
            "config": {"workload": w.name, "kind": w.kind, "n": s.n, "n_targets": n_t, "xi": w.xi, "rc": w.rc,
                       "M": w.M, "P": w.P, "parallelism": f"yslab{world}", "y_split": lay.y_split,
                       "kz_split": lay.kz_split,
                       "l2": "not flushed: each step streams >30 GB of grids/spectra through HBM (126 MB L2)"},
            "e2e": {"value": n_t * args.steps / (ms_e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(bi),
                    "d2h_bytes_per_step": int(hu.numel() * 8), "ms_per_step": ms_e2e / args.steps},
            "gpu_launches": int(launches), "gpu_launches_note": "hand-written kernels only; cuFFT/NCCL excluded",
            "phases_ms_rank0": {k: round(avg[k], 4) for k in ("real", "gridding", "fft", "scale", "ifft", "gather",
                                                              "total")},
            "targets_per_rank": [len(r) for r in rows], "precompute_tables_s": round(t_tables, 3),
            "plan_device_bytes_rank0": st.ev.device_bytes, "clocks": clk}
    if rank == 0:
        emit(line)
    dist.destroy_process_group()


_OUT = None


def emit(line):
    """The one JSON line on the real stdout (fd 1 is redirected to stderr in main(), so NCCL's
    or any library's own stdout chatter cannot interleave with it)."""
    out = _OUT if _OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _OUT
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--workload", default="HL")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="replicas", choices=("replicas", "slab"),
                    help="multi-GPU decomposition: independent replicas (weak) or one y-slab sharded system (strong)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args, rank)
    elif args.mode == "slab":
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        run_slab(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
