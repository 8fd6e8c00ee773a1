#!/bin/bash
# Overlapped tail (tail_overlap_kernel beside a capped ELL grid): parity with
# the mode forced on, then the power-law step over the two grids' CTAs/SM.
set -u
TAG=${1:-ovl}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HEC_TAIL_OVERLAP=1 timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_jacobi.py tests/test_gpu_krylov.py \
    -q > $OUT/pytest_ovl.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_ovl.log
B="python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e --steps 100 --warmup 10"
HEC_TAIL_OVERLAP=0 timeout 300 $B > $OUT/b_off.json 2>> $OUT/err.log
for E in ${OVL_E:-2 3 4}; do
  for T in ${OVL_T:-2 3 4 5}; do
    HEC_TAIL_OVERLAP=1 HEC_OVL_ELL=$E HEC_OVL_TAIL=$T timeout 300 $B > $OUT/b_e${E}_t${T}.json 2>> $OUT/err.log
  done
done
HEC_TAIL_OVERLAP=0 timeout 300 $B > $OUT/b_off2.json 2>> $OUT/err.log
echo done > $OUT/DONE
