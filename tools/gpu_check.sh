# ad-hoc GPU check used during development (run through gpurun); outputs under gpurun_out/$1
set -x
out=gpurun_out/${1:-check}
mkdir -p $out
for v in p0d0 p1d0 p0d1; do
HSEWALD_LIB=$PWD/paper_1802_07844_b200/libhs_$v.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_$v.json 2> $out/bench_$v.err
done
du -sh gpurun_out
