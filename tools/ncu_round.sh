# One GPU call: bench line (no profiler), the launch list of the same command (ncu, per-launch
# times), and full ncu captures (with source) of the hot kernels.  Usage: bash tools/ncu_round.sh TAG
set -x
out=gpurun_out/${1:-ncu}
mkdir -p $out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pair_q|k_gather7|k_spread_mma4|k_xreg|k_mirror_z" \
    -c 6 -o $out/full python tools/profile_step.py --iters 1 > $out/ncu_full.log 2>&1
