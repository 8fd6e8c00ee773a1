#!/bin/bash
# Tail entries per lane with the final tree (HEC_TAIL_EPL 24 / 32 / 48), power-law and degree-sorted, one box,
# alternating.
set -u
OUT=gpurun_out/${1:-epl}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2; do
  for e in 32 24 48; do
    for cfg in powerlaw_8M powerlaw_8M_dsorted; do
      HEC_TAIL_EPL=$e timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_e${e}_$cfg.jsonl 2>> $OUT/err.log
    done
  done
done
echo done > $OUT/DONE
