#!/bin/bash
# Tail entries per lane 48 vs 64 and the tail super-block size (1024 / 2048 / 4096) on the final tree, one box.
set -u
OUT=gpurun_out/${1:-epl2}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2; do
  for v in "48 2048" "64 2048" "48 1024" "48 4096"; do
    set -- $v
    HEC_TAIL_EPL=$1 HEC_TAIL_SUPER=$2 timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_e$1_s$2.jsonl 2>> $OUT/err.log
  done
done
echo done > $OUT/DONE
