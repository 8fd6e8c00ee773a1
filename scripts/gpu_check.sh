#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (N=1), ncu launch list + one full capture.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref.json 2>> $OUT/bench.err
for cfg in poisson3d_128 spe10 powerlaw_8M poisson3d_150; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > $OUT/bench_$cfg.json 2>> $OUT/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv \
  python bench.py --profile --steps 20 --warmup 3 > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ell_kernel -s 5 -c 2 -o $OUT/prof_ell \
  python bench.py --profile --steps 10 --warmup 3 > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
