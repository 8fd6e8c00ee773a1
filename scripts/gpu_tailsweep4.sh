#!/bin/bash
# Paired tail: confirm (MAXLG, EPL) candidates against the default, alternating, two rounds
set -u
OUT=gpurun_out/${1:-tailsweep4}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for r in 1 2; do
  for V in "8 8" "7 10" "7 12" "8 10" "7 8"; do
    set -- $V
    HEC_TAIL_MAXLG=$1 HEC_TAIL_EPL=$2 timeout 300 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e >> $OUT/b_m$1_e$2.jsonl 2>> $OUT/err.log
  done
done
HEC_TAIL_MAXLG=7 timeout 300 python bench.py --config spe10 --no-cpu-baseline --no-e2e >> $OUT/spe10_m7.jsonl 2>> $OUT/err.log
timeout 300 python bench.py --config spe10 --no-cpu-baseline --no-e2e >> $OUT/spe10_m8.jsonl 2>> $OUT/err.log
echo done > $OUT/DONE
