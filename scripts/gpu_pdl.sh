#!/bin/bash
set -u
OUT=gpurun_out/pdl
mkdir -p $OUT
HEC_PDL=1 timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_dist.py -m gpu -q > $OUT/pytest_pdl.log 2>&1; echo "rc=$?" >> $OUT/pytest_pdl.log
for v in "0 1" "1 1" "0 6" "1 6"; do
  set -- $v
  for cfg in poisson3d_256 powerlaw_8M spe10 poisson3d_128; do
    HEC_PDL=$1 HEC_ELL_MINB=$2 timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_pdl$1_minb$2_$cfg.json 2>> $OUT/err.log
  done
done
echo done > $OUT/DONE
