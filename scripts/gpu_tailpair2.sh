#!/bin/bash
# Paired tail loads: unroll / register-cap / entries-per-lane sweep on the power-law step
set -u
OUT=gpurun_out/${1:-tailpair2}; mkdir -p $OUT
run() {  # $1 = tag, $2 = nvcc extra; env passes through
  HEC_NVCC_EXTRA="$2" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
  for cfg in powerlaw_8M spe10; do
    timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$1.json 2>> $OUT/err.log
  done
}
run u1 "-DHEC_TAIL_UNROLL=1"
run u2 ""
run u3 "-DHEC_TAIL_UNROLL=3"
run u2m0 "-DHEC_TAIL_MINB=0"
for E in 4 6 12 16; do HEC_TAIL_EPL=$E run u2e$E ""; done
python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
echo done > $OUT/DONE
