#!/bin/bash
# Quick check of the committed tree: smoke, pytest -m gpu, the default bench line and the tail-heavy lines.
set -u
OUT=gpurun_out/${1:-check}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
for cfg in powerlaw_8M powerlaw_8M_dsorted spe10; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-anchor > $OUT/bench_$cfg.json 2>> $OUT/bench.err
done
echo done > $OUT/DONE
