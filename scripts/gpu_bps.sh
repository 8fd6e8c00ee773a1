#!/bin/bash
set -u
TAG=${1:-r15}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for bps in 0 5 10 15 20 40; do
  for cfg in poisson3d_128 poisson3d_256 spe10; do
    HEC_ELL_BPS=$bps timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_bps${bps}_$cfg.json 2>> $OUT/err.log
  done
done
echo done > $OUT/DONE
