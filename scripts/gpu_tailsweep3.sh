#!/bin/bash
# Paired tail: widest row group (HEC_TAIL_MAXLG) x entries-per-lane target (HEC_TAIL_EPL)
set -u
OUT=gpurun_out/${1:-tailsweep3}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for M in 6 7 8; do for E in 8 10; do
  HEC_TAIL_MAXLG=$M HEC_TAIL_EPL=$E timeout 300 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e > $OUT/b_m${M}_e$E.json 2>> $OUT/err.log
done; done
echo done > $OUT/DONE
