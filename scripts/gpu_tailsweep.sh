#!/bin/bash
set -u
TAG=${1:-r07}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_dist.py -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for run in 8 16; do
  for E in 128 256; do
   HEC_TAIL_RUN=$run HEC_TAIL_E=$E timeout 300 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e --steps 50 > $OUT/pl_r${run}_e${E}.json 2>> $OUT/err.log
  done
done
timeout 300 python bench.py --config spe10 --no-cpu-baseline --no-e2e > $OUT/spe10.json 2>> $OUT/err.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/p256.json 2>> $OUT/err.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 3 -c 1 -o $OUT/prof_tail \
  python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
