# ad-hoc GPU check used during development (run through gpurun); outputs under gpurun_out/$1
set -x
out=gpurun_out/${1:-check}
mkdir -p $out
timeout 1500 python tools/run_configs.py > $out/configs.jsonl 2> $out/configs.err
du -sh gpurun_out
