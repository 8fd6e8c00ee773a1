#!/bin/bash
# Persistent tail grid (HEC_TAIL_PERSIST=1) A/B + parity with it on
set -u
OUT=gpurun_out/${1:-persist2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HEC_TAIL_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_jacobi.py tests/test_gpu_dist.py -q > $OUT/pytest_persist.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_persist.log
for P in 0 1 0 1; do
  for cfg in powerlaw_8M spe10; do
    HEC_TAIL_PERSIST=$P timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e >> $OUT/b_${cfg}_p$P.jsonl 2>> $OUT/err.log
  done
done
echo done > $OUT/DONE
