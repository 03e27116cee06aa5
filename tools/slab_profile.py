"""Per-rank stage costs of the y-slab decomposition, all ranks emulated on ONE GPU
(LocalExchange; ranks run one after another, never waiting on each other).

For each stage, the max over ranks is what one rank of a real W-GPU run would spend on
compute; the exchange volumes are reported so NVLink time can be added (900 GB/s per
direction per GPU).  Usage: python tools/slab_profile.py [workload] [W ...]"""
import json
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_07844_b200 import EwaldParams, ewald_sum  # noqa: E402
from paper_1802_07844_b200.configs import WORKLOADS, make_system  # noqa: E402
from paper_1802_07844_b200.sharding import (LocalExchange, SlabLayout, SlabRank, _partition_targets,  # noqa: E402
                                            _rank_inputs)


def profile(wname, world, reps=3):
    w = WORKLOADS[wname]
    s, targets = make_system(w)
    p = EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P)
    grid = p.grid(s.box_length, s.geometry)
    lay = SlabLayout(grid, world)
    tg, ti, rows = _partition_targets(s, lay, targets, None)
    dev = torch.device("cuda", 0)
    states = [SlabRank(s, p, lay, r, len(rows[r]), device=0) for r in range(world)]
    for st in states:
        st.build_tables()
    inputs = {r: _rank_inputs(s, tg, ti, rows, r, dev) for r in range(world)}
    xch = LocalExchange()
    stages = ("begin", "forward", "kspace", "backward", "finish")
    ms = {k: np.zeros(world) for k in stages}

    def timed(st, name, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for it in range(reps + 1):
        cur = {k: np.zeros(world) for k in stages}
        for st in states:
            cur["begin"][st.rank] = timed(st, "begin", lambda: st.begin(*inputs[st.rank]))
        got = xch.shift(states, "ghost_out", "ghost_in", +1)
        for st in states:
            cur["forward"][st.rank] = timed(st, "forward", lambda: st.forward(st.rank in got))
        xch.all_to_all(states, "send", "recv", lay.fwd_send_splits, lay.fwd_recv_splits)
        for st in states:
            cur["kspace"][st.rank] = timed(st, "kspace", lambda: st.kspace())
        xch.all_to_all(states, "back", "recv_back", lay.fwd_recv_splits, lay.fwd_send_splits)
        for st in states:
            cur["backward"][st.rank] = timed(st, "backward", lambda: st.backward())
        got = xch.shift(states, "halo_out", "halo_in", -1)
        phases = {}
        for st in states:
            res = {}
            cur["finish"][st.rank] = timed(st, "finish", lambda: res.update(st.finish(st.rank in got)))
            phases[st.rank] = res
        if it:
            for k in stages:
                ms[k] += cur[k] / reps
    st0 = states[0]
    a2a_bytes = 8 * (st0.send.numel() + st0.recv_back.numel())   # per rank, both directions
    out = {"workload": wname, "world": world, "y_split": lay.y_split, "kz_split": lay.kz_split,
           "targets_per_rank": [len(r) for r in rows],
           "stage_ms_max": {k: round(float(ms[k].max()), 3) for k in stages},
           "stage_ms_mean": {k: round(float(ms[k].mean()), 3) for k in stages},
           "critical_path_ms": round(float(sum(ms[k].max() for k in stages)), 3),
           "alltoall_bytes_per_rank": int(a2a_bytes * (world - 1) / world),
           "ghost_halo_bytes_per_rank": int(8 * (st0.ghost_out.numel() + st0.halo_out.numel())),
           "plan_bytes_rank0": st0.ev.device_bytes,
           "rank0_phases_ms": {k: round(v, 3) for k, v in phases[0].items()
                               if k in ("real", "gridding", "k_pair", "k_spread", "k_gather", "total")}}
    del states
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    wname = sys.argv[1] if len(sys.argv) > 1 else "HL"
    worlds = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
    for W in worlds:
        print(json.dumps(profile(wname, W)), flush=True)
