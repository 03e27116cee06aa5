# ad-hoc GPU check used during development (run through gpurun); outputs under gpurun_out/$1
set -x
out=gpurun_out/${1:-check}
mkdir -p $out
bash tools/gen_lean_goldens.sh &
gp=$!
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -k "not lean_oracle" > $out/pytest.log 2>&1
bash tools/reference_suite.sh run $out
timeout 600 python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline > $out/bench_cfg5.json 2> $out/bench_cfg5.err
wait $gp
