#!/bin/bash
# Tail L1 eviction hints (HEC_TAIL_L1HINT) A/B on the tail-heavy configs; bench --dist stdout check
set -u
OUT=gpurun_out/${1:-l1hint}; mkdir -p $OUT
for H in 0 1 0 1; do
  HEC_NVCC_EXTRA="-DHEC_TAIL_L1HINT=$H" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
  for cfg in powerlaw_8M spe10; do
    timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e >> $OUT/b_${cfg}_h$H.jsonl 2>> $OUT/err.log
  done
done
python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
timeout 300 python bench.py --dist --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/dist_stdout.txt 2> $OUT/dist_stderr.txt
echo done > $OUT/DONE
