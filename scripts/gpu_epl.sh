#!/bin/bash
set -u
TAG=${1:-r11}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for e in 1 2 4 8; do
  HEC_TAIL_EPL=$e timeout 300 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e --steps 50 > $OUT/pl_epl$e.json 2>> $OUT/err.log
  HEC_TAIL_EPL=$e timeout 300 python bench.py --config spe10 --no-cpu-baseline --no-e2e > $OUT/spe_epl$e.json 2>> $OUT/err.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 3 -c 1 -o $OUT/prof_tail \
  python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
