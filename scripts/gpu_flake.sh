#!/bin/bash
# Flakiness check: the GPU suite three times as the driver runs it (-x), plus smoke
set -u
OUT=gpurun_out/${1:-flake}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for i in 1 2 3; do
  timeout 900 python -m pytest tests/ -x -q -m gpu > $OUT/pytest_$i.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_$i.log
done
echo done > $OUT/DONE
