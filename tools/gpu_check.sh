# ad-hoc GPU check used during development (run through gpurun); outputs under gpurun_out/$1
set -x
out=gpurun_out/${1:-check}
mkdir -p $out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_g8.json 2> $out/bench_g8.err
HSEWALD_LIB=$PWD/paper_1802_07844_b200/libhs_g7.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_g7.json 2> $out/bench_g7.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity.py tests/test_checked_build.py -q -x -k "not lean_oracle" > $out/pytest.log 2>&1
python bench.py --workload cfg2 --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_cfg2.json 2> $out/bench_cfg2.err
du -sh gpurun_out
