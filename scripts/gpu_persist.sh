#!/bin/bash
set -u
TAG=${1:-r09}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_spmv.py -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
HEC_X_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_spmv.py -m gpu -x -q > $OUT/pytest_gpu_persist.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_persist.log
for p in 0 1; do
for cfg in poisson3d_256 powerlaw_8M spe10 poisson3d_128; do
  HEC_X_PERSIST=$p timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_p${p}_$cfg.json 2>> $OUT/err.log
done
done
HEC_X_PERSIST=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 6 -c 6 --csv --log-file $OUT/launches_powerlaw.csv \
    python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > /dev/null 2>&1
echo done > $OUT/DONE
