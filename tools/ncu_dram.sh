# DRAM bytes + duration of ONE kernel of the HL evaluation for the current build and every
# paper_1802_07844_b200/libhs_*.so variant (ncu, two metrics only).  Usage: ncu_dram.sh TAG KERNEL_REGEX
out=gpurun_out/${1:-dram}; kre=${2:-k_spread_mma4}
mkdir -p $out
run() { v=$1; shift
  env "$@" ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"$kre" -c 1 --csv --log-file $out/dram_$v.csv python tools/profile_step.py --iters 1 > $out/dram_$v.log 2>&1
}
run cur HSEWALD_X=0
for f in paper_1802_07844_b200/libhs_*.so; do run $(basename $f .so) HSEWALD_LIB=$PWD/$f; done
