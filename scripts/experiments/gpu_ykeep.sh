#!/bin/bash
# ELL kernel's y store when a big CSR tail follows: streaming (.cs, default) vs plain vs L2 evict_last
# (HEC_Y_KEEP 0/1/2): power-law and degree-sorted step times, per-launch ncu; tail parity on each build.
set -u
OUT=gpurun_out/${1:-yk}
mkdir -p $OUT
for K in 0 1 2; do
  HEC_NVCC_EXTRA="-DHEC_Y_KEEP=$K" python paper_1606_00545_b200/_build.py --force > $OUT/build_$K.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_tail.py -q -p no:cacheprovider > $OUT/pytest_$K.log 2>&1; echo "rc=$?" >> $OUT/pytest_$K.log
  for cfg in powerlaw_8M powerlaw_8M_dsorted; do
    timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_k${K}_$cfg.json 2>> $OUT/err.log
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tail|ell" -c 6 --csv --log-file $OUT/l_k${K}_$cfg.csv \
      python bench.py --config $cfg --profile --steps 3 --warmup 3 > /dev/null 2>&1
  done
done
python paper_1606_00545_b200/_build.py --force > $OUT/build_default.log 2>&1
echo done > $OUT/DONE
