# Generates tests/golden/fullsize_cfg4.npz and fullsize_cfg5.npz with the memory-lean CPU oracle
# on the GPU box's host (196 GB, 16 cores; no GPU used).  Copies them to gpurun_out/ for retrieval.
set -x
mkdir -p gpurun_out/lean_golden
free -g > gpurun_out/lean_golden/host.txt; nproc >> gpurun_out/lean_golden/host.txt
python tests/golden/make_lean_golden.py cfg4 cfg5 > gpurun_out/lean_golden/log.jsonl 2> gpurun_out/lean_golden/err.log
cp tests/golden/fullsize_cfg4.npz tests/golden/fullsize_cfg5.npz gpurun_out/lean_golden/
