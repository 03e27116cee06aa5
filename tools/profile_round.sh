#!/bin/bash
# One GPU call: bench line, launch list of the same command, full ncu captures of the hot kernels.
# Usage (on the GPU box): bash tools/profile_round.sh <tag>
set -u
tag=${1:-r}
out=gpurun_out/$tag
mkdir -p $out
python bench.py --steps 5 --warmup 3 > $out/bench.json 2> $out/bench.err
echo "bench rc=$?" >> $out/status
python bench.py --impl reference --steps 1 --warmup 0 > $out/bench_ref.json 2> $out/bench_ref.err
echo "ref rc=$?" >> $out/status
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_launch.log 2>&1
echo "launch rc=$?" >> $out/status
ncu --set full --clock-control none --import-source on -k regex:"k_pair_q|k_spread_mma|k_mirror_z" -c 4 \
    -o $out/full python tools/profile_step.py --iters 1 > $out/ncu_full.log 2>&1
echo "full rc=$?" >> $out/status
