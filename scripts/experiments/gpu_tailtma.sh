#!/bin/bash
# Tail with the value stream staged by the bulk-copy engine (HEC_TAIL_V 5) x batch x CTAs per SM.
set -u
OUT=gpurun_out/${1:-tt}
mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__throughput.avg.pct_of_peak_sustained_active"
run() {
  local name=$1
  timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-anchor --no-ncu > $OUT/b_$name.json 2>> $OUT/err.log
  timeout 600 ncu --metrics $M --clock-control none -k regex:"tail" -c 2 --csv --log-file $OUT/l_$name.csv python bench.py --config powerlaw_8M --profile --steps 2 --warmup 2 > /dev/null 2>&1
}
first=1
for V in "5 8 6" "5 8 5" "5 6 6" "5 4 8" "4 8 6"; do
  set -- $V
  HEC_NVCC_EXTRA="-DHEC_TAIL_V=$1 -DHEC_TAIL_BATCH=$2 -DHEC_TAIL_MINB=$3" python paper_1606_00545_b200/_build.py --force > $OUT/build_v$1_b$2_m$3.log 2>&1
  if [ $first = 1 ]; then
    timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_fused.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > $OUT/pytest_v5.log 2>&1; echo "rc=$?" >> $OUT/pytest_v5.log
    first=0
  fi
  run v$1_b$2_m$3
done
python paper_1606_00545_b200/_build.py --force > $OUT/build_final.log 2>&1
echo done > $OUT/DONE
