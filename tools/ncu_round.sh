# One GPU call: bench line (no profiler), the launch list of the same command (ncu, per-launch
# times), and full ncu captures (with source) of the hot kernels, summarised ON THE BOX (the
# .ncu-rep files are kept only when small: gpurun copies back at most 64 MiB).
# Usage: bash tools/ncu_round.sh TAG [kernel-regex]
set -x
out=gpurun_out/${1:-ncu}
kre=${2:-"k_pair_q|k_gather7|k_spread_mma4|k_xreg|k_mirror_z"}
mkdir -p $out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$kre" \
    -c 5 -o /tmp/ncu_full python tools/profile_step.py --iters 1 > $out/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/ncu_full.ncu-rep > $out/ncu_summary.json 2>&1
for k in k_pair_q k_gather7 k_spread_mma4 k_xreg; do
  ncu -i /tmp/ncu_full.ncu-rep -k regex:$k --page source --csv --print-source sass > $out/source_$k.csv 2>/dev/null
  gzip -f $out/source_$k.csv
done
ls -la /tmp/ncu_full.ncu-rep >> $out/ncu_full.log
sz=$(stat -c %s /tmp/ncu_full.ncu-rep)
if [ "$sz" -lt 40000000 ]; then cp /tmp/ncu_full.ncu-rep $out/; fi
du -sh gpurun_out
