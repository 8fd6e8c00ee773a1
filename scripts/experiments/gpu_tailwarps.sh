#!/bin/bash
# Tail descriptor size: 8 / 4 / 2 warps per CUDA block (HEC_TAIL_WARPS) x CTAs per SM (HEC_TAIL_MINB):
# power-law, degree-sorted and SPE10 step times, per-launch ncu; parity tests of the 4-warp build.
set -u
OUT=gpurun_out/${1:-tw}
mkdir -p $OUT
run() {  # name, env...
  local name=$1; shift
  for cfg in powerlaw_8M powerlaw_8M_dsorted spe10; do
    env "$@" timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_${name}_$cfg.json 2>> $OUT/err.log
  done
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"tail|ell" -c 6 --csv --log-file $OUT/l_${name}.csv \
     python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
}
for V in "8 6" "4 12" "4 16" "2 24" "2 32"; do
  set -- $V
  HEC_NVCC_EXTRA="-DHEC_TAIL_WARPS=$1 -DHEC_TAIL_MINB=$2" python paper_1606_00545_b200/_build.py --force > $OUT/build_$1_$2.log 2>&1
  if [ "$1 $2" = "4 12" ]; then
    timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_fullsize.py tests/test_gpu_ring.py tests/test_gpu_fused.py -q -p no:cacheprovider > $OUT/pytest_w4.log 2>&1; echo "rc=$?" >> $OUT/pytest_w4.log
  fi
  run w$1_m$2
done
python paper_1606_00545_b200/_build.py --force > $OUT/build_default.log 2>&1
echo done > $OUT/DONE
