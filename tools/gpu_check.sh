# ad-hoc GPU check used during development (run through gpurun); outputs under gpurun_out/$1
set -x
out=gpurun_out/${1:-check}
mkdir -p $out
timeout 900 python -m pytest tests/test_fullsize_parity.py -q -s -k "lean_oracle" > $out/pytest_lean.log 2>&1
timeout 600 python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline > $out/bench_cfg5.json 2> $out/bench_cfg5.err
bash tools/ncu_round.sh ${1:-check}/ncu
du -sh gpurun_out
