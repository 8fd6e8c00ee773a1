#!/bin/bash
# Variant sweep: register vs TMA ELL kernel, stage counts, new tail kernel.
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for K in reg tma; do
  for cfg in poisson3d_256 poisson3d_128 powerlaw_8M spe10 poisson2d_64; do
    HEC_ELL_KERNEL=$K timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_${K}_$cfg.json 2>> $OUT/err.log
  done
done
for S in 2 3 5; do
  HEC_ELL_KERNEL=tma HEC_TMA_STAGES=$S timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/b_tma_s${S}_poisson3d_256.json 2>> $OUT/err.log
done
for K in reg tma; do
  HEC_ELL_KERNEL=$K timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 6 -c 6 --csv --log-file $OUT/launches_${K}_powerlaw.csv \
    python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > /dev/null 2>&1
done
HEC_ELL_KERNEL=tma timeout 900 ncu --set full --clock-control none --import-source on -k regex:ell_tma -s 3 -c 1 -o $OUT/prof_tma \
  python bench.py --profile --steps 5 --warmup 3 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 3 -c 1 -o $OUT/prof_tail \
  python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 >> $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
