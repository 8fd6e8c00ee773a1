#!/bin/bash
set -u
TAG=${1:-r12}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_spmv.py -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for cfg in poisson3d_256 poisson3d_128 powerlaw_8M; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_def_$cfg.json 2>> $OUT/err.log
  for v in 1,0,256 1,1,256 2,0,256 2,1,256 1,0,128 2,1,128; do
    HEC_ELL_X=$v timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_x${v//,/_}_$cfg.json 2>> $OUT/err.log
  done
done
HEC_ELL_X=2,1,256 timeout 900 python -m pytest tests/test_gpu_spmv.py -m gpu -x -q -k "poisson or powerlaw" > $OUT/pytest_x.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_x.log
echo done > $OUT/DONE
