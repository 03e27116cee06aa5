# compute-sanitizer memcheck and racecheck (and synccheck) over tools/sanitize_case.py.
# Usage (GPU box): bash tools/sanitize.sh OUTDIR [N]
set -x
out=${1:-gpurun_out/sanitize}
n=${2:-3000}
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_case.py $n > $out/plain.log 2>&1
timeout 1800 $CS --tool memcheck --leak-check no --report-api-errors no --print-limit 50 \
    python tools/sanitize_case.py $n > $out/memcheck.log 2>&1
echo "memcheck rc=$?" >> $out/memcheck.log
timeout 2400 $CS --tool racecheck --racecheck-report hazard --print-limit 50 \
    python tools/sanitize_case.py 1500 > $out/racecheck.log 2>&1
echo "racecheck rc=$?" >> $out/racecheck.log
timeout 1800 $CS --tool synccheck --print-limit 50 python tools/sanitize_case.py 1500 > $out/synccheck.log 2>&1
echo "synccheck rc=$?" >> $out/synccheck.log
