# A/B of library variants on one GPU box (run through gpurun): optional pytest selection, then
# the HL bench line for every paper_1802_07844_b200/libhs_*.so variant and the current build.
# Usage: bash tools/ab.sh TAG ["pytest -k expression"]
set -x
out=gpurun_out/${1:-ab}
mkdir -p $out
if [ -n "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$2" > $out/pytest.log 2>&1
  echo "pytest rc=$?" >> $out/pytest.log
fi
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_new.json 2> $out/bench_new.err
for f in paper_1802_07844_b200/libhs_*.so; do
  v=$(basename $f .so)
  HSEWALD_LIB=$PWD/$f python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_$v.json 2> $out/bench_$v.err
done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_new2.json 2> $out/bench_new2.err
