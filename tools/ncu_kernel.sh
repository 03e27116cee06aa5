# ncu --set full (with source) of ONE kernel of the HL evaluation, for the current build and every
# paper_1802_07844_b200/libhs_*.so variant; summaries + SASS source pages under gpurun_out/$1.
# Usage: bash tools/ncu_kernel.sh TAG KERNEL_REGEX
set -x
out=gpurun_out/${1:-ncuk}
kre=${2:-k_pair_q}
mkdir -p $out
python tools/profile_step.py --iters 1 > $out/plain.log 2>&1 || exit 1
run() {  # $1 = variant name, rest = env
  v=$1; shift
  env "$@" ncu -f --set full --clock-control none --import-source on -k regex:"$kre" -c 1 \
      -o /tmp/ncu_$v python tools/profile_step.py --iters 1 > $out/ncu_$v.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$v.ncu-rep > $out/summary_$v.json 2>&1
  ncu -i /tmp/ncu_$v.ncu-rep --page source --csv --print-source sass > $out/source_$v.csv 2>/dev/null
  gzip -f $out/source_$v.csv
}
run cur HSEWALD_X=0
for f in paper_1802_07844_b200/libhs_*.so; do
  v=$(basename $f .so)
  run $v HSEWALD_LIB=$PWD/$f
done
du -sh $out
