# The round-end driver's commands on one GPU box, plus the profiling set; outputs under
# gpurun_out/$1 (copied into profiles/ afterwards).  Usage: bash tools/final_round.sh TAG
set -x
out=gpurun_out/${1:-final}
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/gpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke.log 2>&1
echo "smoke rc=$?" >> $out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $out/pytest_gpu.log
python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $out/bench_ref.json 2> $out/bench_ref.err
bash tools/reference_suite.sh run $out
bash tools/ncu_round.sh ${1:-final}/ncu
du -sh gpurun_out
