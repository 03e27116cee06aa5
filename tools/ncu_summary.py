"""Summarise an ncu report (raw page) into the metrics we track per kernel."""
import csv
import io
import subprocess
import sys

METRICS = [
    ("time_ms", "gpu__time_duration.sum"),
    ("regs", "launch__registers_per_thread"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("fp64_pipe_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    ("dram_read_MB", "dram__bytes_read.sum"),
    ("dram_write_MB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l1tex_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("l2_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("smem_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("thread_inst_per_inst", "smsp__thread_inst_executed_per_inst_executed.ratio"),
    ("inst_executed", "smsp__inst_executed.sum"),
]
STALLS = ["barrier", "short_scoreboard", "long_scoreboard", "math_pipe_throttle", "wait", "mio_throttle",
          "lg_throttle", "no_instruction", "not_selected", "selected", "dispatch_stall", "branch_resolving",
          "membar", "sleeping", "drain", "imc_miss", "tex_throttle", "misc"]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:70]}
        for k, m in METRICS:
            if m in h:
                d[k] = r[h.index(m)] + ("" if not units[h.index(m)] else " " + units[h.index(m)])
        stall = {}
        for s in STALLS:
            m = f"smsp__average_warp_latency_issue_stalled_{s}.ratio"
            m2 = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            for mm in (m2, m):
                if mm in h:
                    try:
                        stall[s] = float(r[h.index(mm)])
                    except ValueError:
                        pass
                    break
        if stall:
            d["stalls_per_issue"] = {k: round(v, 3) for k, v in sorted(stall.items(), key=lambda x: -x[1])[:6]}
        out.append(d)
    return out


if __name__ == "__main__":
    import json
    for d in summarise(sys.argv[1]):
        print(json.dumps(d, indent=1))
