#!/usr/bin/env python
"""Headline benchmark: half-space stokeslet Ewald target evaluations/s at N=1e6, FP64
(BASELINE.json `metric`, workload "HL": N=1e6, xi=49.92, r_c=0.101, M=192, P=24).

One step = one full ewald_sum evaluation (real + Fourier) of the whole system,
inputs resident in HBM, Green's tables precomputed outside the timed region (as
the reference and the paper do).  `e2e` repeats the measurement through the
C ABI with pinned HOST buffers (H2D of positions+strengths(+targets) and D2H of
velocities inside the timed region).  `cpu_baseline` and `--impl reference`
time COMPLETE evaluations of the same workload by the CPU restatement of the
reference (oracle/, C + OpenMP + scipy.fft) on all host cores.

--workload: HL (default, the metric's configuration), cfg1..cfg5 (cfg5: the mixed
stokeslet + stresslet system with separate targets).

Multi-GPU (torchrun, or --gpus N which launches the N ranks itself):
  --mode slab (default for N > 1): ONE system y-slab decomposed over the ranks
      (sharding.py: spread ghost planes, per-channel NCCL all-to-all transposes of
      the FFT, gather halo; strong scaling, value = N_targets / time of one sharded
      evaluation, max over ranks);
  --mode replicas: every rank evaluates its own independent system (weak scaling,
      no data-path collective).
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
# CPU baseline: the oracle port (test infrastructure; oracle/), one FULL evaluation timed
FULL_COMPLEX_MAX = 400_000_000   # padded grid points up to which the port keeps the reference's full
                                 # complex spectra (ref:ewald_fourier.py:518-532); above: R2C lean mode


def cpu_tables(wname, threads):
    """Green's tables for the port (precompute excluded from the timing, as in the reference)."""
    from oracle import hsoracle as o
    from paper_1802_07844_b200.configs import WORKLOADS
    w = WORKLOADS[wname]
    g = o.Grid(w.L, w.M, w.P, w.xi, "half")
    kinds = ["stokeslet", "stresslet"] if w.kind == "mixed" else [w.kind]
    need = sorted(set(sum((o.table_kinds_for(k, "half") for k in kinds), [])))
    half = {k: o.precompute_greens_half(k, g, workers=threads) for k in need}
    full = None
    if int(np.prod(g.padded_dims)) <= FULL_COMPLEX_MAX:
        full = {k: o.expand_half_table(v, g.padded_dims) for k, v in half.items()}
    return g, half, full


def cpu_full_eval(wname, threads, tabs):
    """Seconds for ONE complete ewald_sum evaluation of the workload by the port on `threads` host
    cores: real space at every target, every source spread, every transform, every gather.
    Mixed workloads: the reference's two calls (one per kind)."""
    from oracle import hsoracle as o
    from paper_1802_07844_b200.configs import WORKLOADS, make_system
    w = WORKLOADS[wname]
    o.set_threads(threads)
    s, tg = make_system(w)
    g, half, full = tabs
    systems = [("stokeslet", s.stokeslet), ("stresslet", s.stresslet)] if w.kind == "mixed" else [(w.kind, s)]
    t0 = time.perf_counter()
    for kind, ps in systems:
        kw = {"f": ps.f} if kind == "stokeslet" else {"g": ps.g, "q": ps.q}
        if full is not None:
            o.ewald_sum(kind, "half", w.L, ps.positions, w.xi, w.rc, w.M, w.P, full, targets=tg, workers=threads,
                        **kw)
        else:
            o.ewald_sum_lean(kind, "half", w.L, ps.positions, w.xi, w.rc, w.M, w.P, half, targets=tg,
                             workers=threads, **kw)
    t = time.perf_counter() - t0
    mode = "full complex spectra (the reference's layout)" if full is not None else "R2C lean mode"
    nt = s.n if tg is None else tg.shape[0]
    desc = (f"oracle port (C + OpenMP, scipy.fft; {threads} threads): one complete evaluation of {wname} "
            f"(N={s.n}, {nt} targets, padded {tuple(g.padded_dims)}, {mode}); tables precomputed outside the "
            f"timed region")
    return t, desc, nt


def cpu_host():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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


def config_of(w):
    """The `config` both arms print (identical keys, so the driver's same_config holds)."""
    return {"workload": w.name, "kind": w.kind, "n": w.n, "n_targets": w.n, "L": w.L, "xi": w.xi, "rc": w.rc,
            "M": w.M, "P": w.P}


def run_reference(args, rank):
    """The reference arm: the port on all host cores.  W warm-up evaluations of the small cfg1
    system (thread pools, FFT plans), then complete evaluations of the workload, best of up to
    `steps` (best of 3) within a ~3 minute budget; `steps` = evaluations
    actually timed."""
    if rank != 0:
        return
    from paper_1802_07844_b200.configs import WORKLOADS
    w = WORKLOADS[args.workload]
    thr = os.cpu_count()
    t_tab0 = time.perf_counter()
    tabs = cpu_tables(args.workload, thr)
    t_tab = time.perf_counter() - t_tab0
    small = cpu_tables("cfg1", thr)
    for _ in range(args.warmup):
        cpu_full_eval("cfg1", thr, small)
    times = []
    t_start = time.perf_counter()
    while len(times) < max(1, args.steps):
        t, desc, nt = cpu_full_eval(args.workload, thr, tabs)
        times.append(t)
        if time.perf_counter() - t_start + t > args.ref_budget_s:
            break
    best = min(times)
    value = nt / best
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": len(times),
            "warmup": args.warmup, "ms_per_step": best * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded PCG64, BASELINE.json shapes)",
            "config": config_of(w), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "port", "sample": desc,
                             "host": cpu_host(), "timed_evaluations_s": [round(x, 3) for x in times],
                             "statistic": f"best of {len(times)}", "tables_s": round(t_tab, 2),
                             "requested_steps": args.steps},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


PAIR_INSTR = {"stokeslet": (64, 33), "stresslet": (85, 50), "rotlet": (62, 28), "mixed": (64 + 85, 33 + 50)}


def run_ours(args, rank, world, local_rank):
    """One plan per rank: N = 1, or N independent replicas (--mode replicas, weak scaling)."""
    import torch
    import torch.distributed as dist
    from paper_1802_07844_b200 import GridSpec, _lib
    from paper_1802_07844_b200._plan import Evaluator
    from paper_1802_07844_b200.configs import WORKLOADS, Workload, make_system
    from paper_1802_07844_b200.ewald import _strengths

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    w0 = WORKLOADS[args.workload]
    w = Workload(**{**w0.__dict__, "seed": w0.seed + 7919 * rank})   # replicas: independent systems
    s, targets = make_system(w)
    nt = s.n if targets is None else targets.shape[0]
    grid = GridSpec(L=w.L, M=w.M, P=w.P, xi=w.xi, geometry="half")
    ev = Evaluator(w.kind, "half", w.L, w.xi, w.rc, grid, s.n, nt, targets is None, device=local_rank)
    t0 = time.perf_counter()
    ev.build_tables()
    t_tables = time.perf_counter() - t0
    dev = torch.device("cuda", local_rank)
    fa, fb = _strengths(s)
    host_in = [np.ascontiguousarray(a, dtype=np.float64) for a in (s.positions, fa, fb, targets) if a is not None]
    dput = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)  # noqa: E731
    pos, sa, sb, tgd = dput(s.positions), dput(fa), dput(fb), dput(targets)
    out = torch.empty((3, nt, 3), dtype=torch.float64, device=dev)
    run = lambda what=3: ev.execute(pos, sa, sb, targets=tgd, out=out, what=what)  # noqa: E731
    for _ in range(args.warmup):
        run()
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
    for _ in range(args.steps):
        run()
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
    step_times = [run(7)[3] for _ in range(args.steps)]
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    value = world * nt * args.steps / (ms * 1e-3)
    avg = {k: float(np.mean([t[k] for t in step_times])) for k in step_times[0]}

    # ---- e2e through the C ABI with pinned host buffers (inputs H2D and velocities D2H every step)
    pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
    hin = [pin(a) for a in host_in]
    hu = torch.empty((nt, 3), dtype=torch.float64).pin_memory()
    hv = [t.numpy() for t in hin]
    hpos, hfa = hv[0], hv[1]
    hfb = hv[2] if fb is not None else None
    htg = hv[-1] if targets is not None else None
    hout = hu.numpy()
    ev.execute(hpos, hfa, hfb, targets=htg, out=(hout, None, None))   # warm
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        ev.execute(hpos, hfa, hfb, targets=htg, out=(hout, None, None))
    e1.record()
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_e2e = float(tt.item())
    e2e_value = world * nt * args.steps / (ms_e2e * 1e-3)
    e2e_consistent = bool(np.array_equal(out[0].cpu().numpy(), hout))

    # ---- roofline (algorithmic work per launch)
    hbm_peak, fp64_peak, peak_src = _peaks()
    P3 = w.P ** 3
    n_in, n_out = ev.fft_counts()
    n_half = grid.padded_dims[0] * grid.padded_dims[1] * (grid.padded_dims[2] // 2 + 1)
    pairs, img_pairs = avg["pairs"], avg["image_pairs"]
    pi, pc = PAIR_INSTR[w.kind]
    work = {
        # mirrored spreading (csrc/plan.cu k_mirror_z): kernel + wall channels at the N sources,
        # images by reflection of the grid (stokeslet: 10 N P^3 -> 7 N P^3 FMAs)
        "k_spread": ("flop", 2.0 * P3 * n_in * s.n, "fp64:dmma"),
        # k_gather8: the z contraction on the FP64 tensor pipe (DMMA)
        "k_gather": ("flop", 2.0 * P3 * n_out * nt, "fp64:dmma"),
        "k_scale": ("bytes", n_half * (16 * n_in + 16 * n_out + 8 * 2), "hbm"),
        "k_pair": ("flop", 2.0 * (pi * pairs + pc * img_pairs), "fp64:dfma"),
    }
    kern = roofline(avg, work, hbm_peak, fp64_peak)
    dom = max(kern, key=lambda k: kern[k]["ms"])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_per_launch.json")
    if os.path.exists(tp) and w.name == "HL":
        traffic = json.load(open(tp)).get(dom)
    rf = dict(kern[dom])
    rf.update({"kernel": dom, "traffic": traffic, "peak_source": (
        "MEASURED_PEAKS.json hbm_gbs" if rf["bound"] == "hbm" else
        f"measured FP64 {rf['pipe'].upper()} microbenchmark, profiles/r01_probe_fp64.json")})

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded PCG64, BASELINE.json shapes)",
            "config": config_of(w),
            "run": {"padded_dims": list(grid.padded_dims), "parallelism": f"replicas{world}",
                    "streams": "real space concurrent with the Fourier pipeline up to the gather; "
                               "kernels/phases_ms/roofline from the same steps run serialised",
                    "l2": "not flushed: each step streams >30 GB of grids/spectra through HBM (126 MB L2)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(sum(t.numel() * 8 for t in hin)),
                    "d2h_bytes_per_step": int(hu.numel() * 8), "ms_per_step": ms_e2e / args.steps,
                    "matches_device_result": e2e_consistent},
            "gpu_launches": int(launches), "gpu_launches_note": "hand-written kernels only; cuFFT launches excluded",
            "roofline": rf, "kernels": kern,
            "phases_ms": {k: round(avg[k], 4) for k in ("real", "gridding", "fft", "scale", "ifft", "gather",
                                                        "total")},
            "pairs_per_step": pairs, "image_pairs_per_step": img_pairs, "fft_count_executed": [n_in, n_out],
            "precompute_tables_s": round(t_tables, 3), "plan_device_bytes": ev.device_bytes,
            "clocks": clk}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr = os.cpu_count()
        t0 = time.perf_counter()
        tabs = cpu_tables(args.workload, thr)
        t_tab = time.perf_counter() - t0
        t, desc, nt_c = cpu_full_eval(args.workload, thr, tabs)
        line["cpu_baseline"] = {"value": nt_c / t, "unit": UNIT, "cores": thr, "kind": "port", "sample": desc,
                                "host": cpu_host(), "timed_evaluations_s": [round(t, 3)], "tables_s": round(t_tab, 2)}
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
    # one GPU per rank: NCCL over NVLink.  Ranks sharing one GPU (bench.py --gpus N on a smaller
    # lease): gloo with host-staged exchanges -- a functional run of the sharded path, not a
    # scaling measurement (no kernel waits on another rank, so sharing the device is safe)
    backend = os.environ.get("HS_BENCH_BACKEND", "nccl")
    dist.init_process_group(backend, device_id=dev if backend == "nccl" else None, rank=rank, world_size=world)
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
            "config": config_of(w),
            "run": {"parallelism": f"yslab{world}", "exchange": backend + ("" if backend == "nccl" else
                                                                            " (host-staged; ranks share a GPU)"),
                    "y_split": lay.y_split, "kz_split": lay.kz_split,
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
    ap.add_argument("--mode", default=None, choices=("replicas", "slab"),
                    help="multi-GPU decomposition: one y-slab sharded system (strong scaling; default for N > 1) "
                         "or independent replicas (weak scaling)")
    ap.add_argument("--ref-budget-s", type=float, default=180.0,
                    help="reference arm: stop timing further full evaluations after this many seconds")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    mode = args.mode or ("slab" if world > 1 else "replicas")
    if mode == "slab":
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        run_slab(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


def spawn_ranks(args):
    """bench.py --gpus N without torchrun: launch the N ranks here (one process per GPU, NCCL;
    with fewer visible GPUs than N the ranks share GPU 0 over gloo with host-staged exchanges).
    Rank 0's JSON line is forwarded; returns the worst exit code."""
    import socket
    import torch
    ngpu = torch.cuda.device_count()
    share = ngpu < args.gpus
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(args.gpus), LOCAL_RANK=str(0 if share else r),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   HS_BENCH_BACKEND="gloo" if share else "nccl")
        if not share:
            env.setdefault("NCCL_DEBUG", "INFO")   # communicator set-up (NVLink / NVLS) on stderr
        procs.append(subprocess.Popen([sys.executable] + sys.argv, env=env, stdout=subprocess.PIPE,
                                      stderr=None, text=True))
    outs = [p.communicate()[0] for p in procs]
    for ln in outs[0].splitlines():
        if ln.strip():
            emit(json.loads(ln))
    return max(p.returncode for p in procs)


if __name__ == "__main__":
    main()
