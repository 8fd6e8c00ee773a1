#!/bin/bash
# Power-law ELL width sweep (FIXED policy) with the paired-load tail
set -u
OUT=gpurun_out/${1:-width2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for W in 7 8 9 10 11 12; do
  timeout 300 python bench.py --config powerlaw_8M --ell-width $W --no-cpu-baseline --no-e2e > $OUT/b_powerlaw_8M_w$W.json 2>> $OUT/err.log
done
echo done > $OUT/DONE
