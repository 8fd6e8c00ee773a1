#!/bin/bash
OUT=gpurun_out/phase
mkdir -p $OUT
for ph in 16 8 6; do
  HEC_NVCC_EXTRA="-DHEC_ELL_PHASE=$ph" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" > $OUT/build_$ph.log 2>&1
  for cfg in powerlaw_8M poisson3d_256 spe10 poisson3d_128; do
    echo "== $ph $cfg" >> $OUT/bench.jsonl
    timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 200 --warmup 20 >> $OUT/bench.jsonl 2>> $OUT/bench.err
  done
done
HEC_NVCC_EXTRA="-DHEC_ELL_PHASE=8" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)"
timeout 600 python -m pytest tests/test_gpu_spmv.py -q -x -p no:cacheprovider > $OUT/pytest8.log 2>&1; echo "rc=$?" >> $OUT/pytest8.log
