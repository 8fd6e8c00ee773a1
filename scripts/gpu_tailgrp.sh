#!/bin/bash
set -u
OUT=gpurun_out/tailgrp
mkdir -p $OUT
HEC_TAIL=group timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_dist.py tests/test_gpu_krylov.py -m gpu -q > $OUT/pytest_group.log 2>&1; echo "rc=$?" >> $OUT/pytest_group.log
for t in bins group; do
  for cfg in powerlaw_8M spe10; do
    HEC_TAIL=$t timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_${t}_$cfg.json 2>> $OUT/err.log
  done
done
HEC_TAIL=group timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 9 -c 9 --csv --log-file $OUT/launches_group_powerlaw.csv \
    python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > /dev/null 2>&1
echo done > $OUT/DONE
