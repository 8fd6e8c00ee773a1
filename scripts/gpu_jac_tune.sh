#!/bin/bash
OUT=gpurun_out/jac_tune
mkdir -p $OUT
for mb in 0 5 4; do
  HEC_NVCC_EXTRA="-DHEC_JAC_MINB=$mb" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" > $OUT/build_$mb.log 2>&1
  for cfg in poisson3d_256 powerlaw_8M spe10; do
    echo "minb=$mb" >> $OUT/bench.jsonl
    timeout 600 python bench.py --jacobi 0.8 --config $cfg --steps 100 --warmup 5 >> $OUT/bench.jsonl 2>> $OUT/bench.err
  done
done
python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)"
timeout 600 python -m pytest tests/test_gpu_jacobi.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
