#!/bin/bash
# Tail descriptor order chosen per matrix (reverse unless heavy descriptors lead): parity + default lines.
set -u
OUT=gpurun_out/${1:-rev2}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tail.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do
  for cfg in powerlaw_8M powerlaw_8M_dsorted spe10; do
    timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_$cfg.jsonl 2>> $OUT/err.log
  done
done
echo done > $OUT/DONE
