#!/bin/bash
# Power-law ELL width sweep (FIXED policy) with the round-2 tail: does the BG3 width (reading A1) stay best?
set -u
OUT=gpurun_out/${1:-wd}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for w in 6 7 8 9 10 11 12; do
  timeout 600 python bench.py --config powerlaw_8M --ell-width $w --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-anchor > $OUT/b_w$w.json 2>> $OUT/err.log
done
timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-anchor --no-ncu > $OUT/b_bg3.json 2>> $OUT/err.log
echo done > $OUT/DONE
