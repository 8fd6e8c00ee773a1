#!/bin/bash
set -u
OUT=gpurun_out/${1:-q2}
mkdir -p $OUT
for p in 0 1; do
for cfg in poisson3d_256 powerlaw_8M spe10 poisson3d_128; do
  HEC_PDL=$p timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_pdl${p}_$cfg.json 2>> $OUT/err.log
done
done
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_spmv.py -m gpu -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
echo done > $OUT/DONE
