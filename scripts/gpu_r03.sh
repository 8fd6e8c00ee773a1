#!/bin/bash
set -u
TAG=${1:-r03}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for cfg in poisson3d_256 powerlaw_8M spe10 poisson3d_128; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline > $OUT/b_$cfg.json 2>> $OUT/err.log
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 6 -c 6 --csv --log-file $OUT/launches_powerlaw.csv \
    python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 3 -c 1 -o $OUT/prof_tail \
  python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
