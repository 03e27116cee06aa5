# ad-hoc GPU check used during development (run through gpurun); outputs under gpurun_out/$1
set -x
out=gpurun_out/${1:-check}
mkdir -p $out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_m1.json 2> $out/bench_m1.err
HSEWALD_LIB=$PWD/paper_1802_07844_b200/libhs_m0.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_m0.json 2> $out/bench_m0.err
timeout 900 python -m pytest tests/test_fullsize_parity.py tests/test_checked_build.py tests/test_gpu_parity.py -q -x -k "not lean_oracle" > $out/pytest.log 2>&1
python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_cfg3.json 2> $out/bench_cfg3.err
du -sh gpurun_out
