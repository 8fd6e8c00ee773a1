#!/bin/bash
# ELL CTA size (HEC_ELL_BLOCK) on the small and large configs
set -u
OUT=gpurun_out/${1:-ellblock}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for r in 1 2; do
  for B in 256 128; do
    for cfg in spe10 poisson3d_128 poisson3d_256 powerlaw_8M; do
      HEC_ELL_BLOCK=$B timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 100 --warmup 10 >> $OUT/b_${cfg}_b$B.jsonl 2>> $OUT/err.log
    done
  done
done
HEC_ELL_BLOCK=128 timeout 600 python -m pytest tests/test_gpu_spmv.py -q -x > $OUT/pytest_b128.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_b128.log
echo done > $OUT/DONE
