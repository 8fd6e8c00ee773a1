#!/bin/bash
# Tail chunk size sweep (HEC_TAIL_U): parity at the default, power-law + SPE10 step per U
set -u
OUT=gpurun_out/${1:-tailu}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_jacobi.py tests/test_gpu_dist.py -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for U in ${TAIL_US:-8 4 6 12}; do
  HEC_NVCC_EXTRA="-DHEC_TAIL_U=$U" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
  for cfg in powerlaw_8M spe10; do
    timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_u$U.json 2>> $OUT/err.log
  done
done
echo done > $OUT/DONE
