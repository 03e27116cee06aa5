# ad-hoc GPU check used during development (run through gpurun); outputs under gpurun_out/$1
set -x
out=gpurun_out/${1:-check}
mkdir -p $out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_a.json 2> $out/bench_a.err
HSEWALD_LIB=$PWD/paper_1802_07844_b200/libhs_n1.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_n1.json 2> $out/bench_n1.err
HSEWALD_LIB=$PWD/paper_1802_07844_b200/libhs_n1.so timeout 900 python -m pytest tests/test_fullsize_parity.py -q -s -k "vs_reference" > $out/pytest_n1.log 2>&1
timeout 900 python -m pytest tests/test_fullsize_parity.py -q -s -k "vs_reference" > $out/pytest_a.log 2>&1
du -sh gpurun_out
