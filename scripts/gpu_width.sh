#!/bin/bash
OUT=gpurun_out/width
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for w in 9 10 11 12 14 16; do
  echo "== w $w" >> $OUT/bench.jsonl
  timeout 600 python bench.py --config powerlaw_8M --ell-width $w --no-cpu-baseline --no-e2e --steps 100 --warmup 10 >> $OUT/bench.jsonl 2>> $OUT/bench.err
done
