#!/bin/bash
# ELL first/second phase split for two-phase widths (HEC_ELL_P1_DELTA -1 / 0 / +1; W = 9: 4+5, 5+4, 6+3 slots)
# with slot skipping and grouping: power-law and degree-sorted step times on one box, alternating.
set -u
OUT=gpurun_out/${1:-p1}
mkdir -p $OUT
for i in 1 2; do
  for D in -1 0 1; do
    HEC_NVCC_EXTRA="-DHEC_ELL_P1_DELTA=$D" python paper_1606_00545_b200/_build.py --force > $OUT/build_$D.log 2>&1
    for cfg in powerlaw_8M powerlaw_8M_dsorted; do
      timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_d${D}_$cfg.jsonl 2>> $OUT/err.log
    done
  done
done
HEC_NVCC_EXTRA="-DHEC_ELL_P1_DELTA=-1" python paper_1606_00545_b200/_build.py --force > $OUT/build_t.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tileskip.py -q -p no:cacheprovider > $OUT/pytest_dm1.log 2>&1; echo "rc=$?" >> $OUT/pytest_dm1.log
python paper_1606_00545_b200/_build.py --force > $OUT/build_default.log 2>&1
echo done > $OUT/DONE
