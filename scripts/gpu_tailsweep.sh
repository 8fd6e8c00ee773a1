#!/bin/bash
set -u
TAG=${1:-r06}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_dist.py -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for keep in 0 1; do
 for run in 8 16; do
  for E in 256 512; do
   HEC_X_KEEP=$keep HEC_TAIL_RUN=$run HEC_TAIL_E=$E timeout 300 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e --steps 50 > $OUT/pl_k${keep}_r${run}_e${E}.json 2>> $OUT/err.log
  done
 done
 HEC_X_KEEP=$keep timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/p256_k${keep}.json 2>> $OUT/err.log
 HEC_X_KEEP=$keep timeout 300 python bench.py --config spe10 --no-cpu-baseline --no-e2e > $OUT/spe10_k${keep}.json 2>> $OUT/err.log
done
echo done > $OUT/DONE
