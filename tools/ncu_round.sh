# One GPU call: bench line (no profiler), the launch list of the same command (ncu, per-launch
# times), and one full ncu capture (with SASS source page) per hot kernel, summarised ON THE BOX.
# Usage: bash tools/ncu_round.sh TAG [kernel names...]
set -x
out=gpurun_out/${1:-ncu}; shift
ks=${@:-"k_pair_q k_spread_mma4 k_gather8 k_xreg k_zfwd k_zinv k_ystage"}
mkdir -p $out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_launch.log 2>&1
python tools/profile_step.py --iters 1 > $out/plain.log 2>&1 || exit 1
: > $out/ncu_summary.json
for k in $ks; do
  ncu -f --set full --clock-control none --import-source on -k regex:"$k" -c 1 -o /tmp/ncu_$k \
      python tools/profile_step.py --iters 1 > $out/ncu_$k.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$k.ncu-rep >> $out/ncu_summary.json 2>&1
  ncu -i /tmp/ncu_$k.ncu-rep --page source --csv --print-source sass > $out/source_$k.csv 2>/dev/null
  gzip -f $out/source_$k.csv
done
du -sh gpurun_out
