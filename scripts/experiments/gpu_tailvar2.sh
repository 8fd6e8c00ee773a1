#!/bin/bash
# Tail kernel sweep 2: entries per lane x (plain unroll 2 | batched loads of 4 / 8 iterations, CTAs per SM).
set -u
OUT=gpurun_out/${1:-tv2}
mkdir -p $OUT
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_$name.json 2>> $OUT/err.log
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"tail" -c 3 --csv --log-file $OUT/l_$name.csv \
     python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
}
for V in "0 2 4 8" "4 2 4 8" "4 2 8 8" "4 2 8 6" "4 2 8 4"; do
  set -- $V
  HEC_NVCC_EXTRA="-DHEC_TAIL_V=$1 -DHEC_TAIL_UNROLL=$2 -DHEC_TAIL_BATCH=$3 -DHEC_TAIL_MINB=$4" python paper_1606_00545_b200/_build.py --force > $OUT/build_v$1_b$3_m$4.log 2>&1
  for epl in 8 16 32; do
    run v$1_b$3_m$4_epl$epl HEC_TAIL_WIN=0 HEC_TAIL_EPL=$epl
  done
done
echo done > $OUT/DONE
