#!/bin/bash
# GPU tests + tail-heavy bench lines (power-law, SPE10) + 256^3
set -u
OUT=gpurun_out/${1:-rq4}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for cfg in powerlaw_8M spe10 poisson3d_256; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_$cfg.json 2>> $OUT/err.log
done
timeout 300 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e --jacobi 0.8 > $OUT/b_powerlaw_jacobi.json 2>> $OUT/err.log
echo done > $OUT/DONE
