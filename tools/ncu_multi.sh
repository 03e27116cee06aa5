# ncu --set full (with SASS source pages) of several kernels of one HL evaluation of the current build.
# Usage: bash tools/ncu_multi.sh TAG KERNEL_REGEX [KERNEL_REGEX ...]
set -x
out=gpurun_out/${1:-ncum}; shift
mkdir -p $out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
python tools/profile_step.py --iters 1 > $out/plain.log 2>&1 || exit 1
for kre in "$@"; do
  v=$(echo $kre | tr -c 'A-Za-z0-9_\n' '_')
  ncu -f --set full --clock-control none --import-source on -k regex:"$kre" -c 1 \
      -o /tmp/ncu_$v python tools/profile_step.py --iters 1 > $out/ncu_$v.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$v.ncu-rep > $out/summary_$v.json 2>&1
  ncu -i /tmp/ncu_$v.ncu-rep --page source --csv --print-source sass > $out/source_$v.csv 2>/dev/null
  gzip -f $out/source_$v.csv
done
du -sh $out
