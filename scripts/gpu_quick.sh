#!/bin/bash
# tests + bench lines for the main configs + launch list of the power-law step
set -u
TAG=${1:-rq}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for cfg in poisson3d_256 powerlaw_8M spe10 poisson3d_128; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline > $OUT/b_$cfg.json 2>> $OUT/err.log
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 6 -c 6 --csv --log-file $OUT/launches_powerlaw.csv \
    python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > /dev/null 2>&1
echo done > $OUT/DONE
