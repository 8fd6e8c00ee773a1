#!/bin/bash
# Tail vector width 4 (quads): GPU parity with it, then power-law / SPE10 at unroll 1/2
set -u
OUT=gpurun_out/${1:-tailvec}; mkdir -p $OUT
HEC_NVCC_EXTRA="-DHEC_TAIL_VEC=4" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_jacobi.py tests/test_gpu_dist.py tests/test_gpu_p2p.py -q > $OUT/pytest_vec4.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_vec4.log
run() {
  HEC_NVCC_EXTRA="$2" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
  for cfg in powerlaw_8M spe10; do
    timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$1.json 2>> $OUT/err.log
  done
}
run v4u1 "-DHEC_TAIL_VEC=4 -DHEC_TAIL_UNROLL=1"
run v4u2 "-DHEC_TAIL_VEC=4 -DHEC_TAIL_UNROLL=2"
run v2u2 ""
python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
echo done > $OUT/DONE
