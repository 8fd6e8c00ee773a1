#!/bin/bash
# Paired tail loads (even-padded rows): GPU parity, then power-law / SPE10 under
# register caps and unroll depths
set -u
OUT=gpurun_out/${1:-tailpair}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for V in "-DHEC_TAIL_MINB=8" "-DHEC_TAIL_MINB=0" "-DHEC_TAIL_MINB=8 -DHEC_TAIL_UNROLL=2" "-DHEC_TAIL_MINB=8 -DHEC_TAIL_UNROLL=8"; do
  TAGV=$(echo "$V" | tr -d ' =-' )
  HEC_NVCC_EXTRA="$V" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
  for cfg in powerlaw_8M spe10; do
    timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $OUT/b_${cfg}_$TAGV.json 2>> $OUT/err.log
  done
done
python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
timeout 300 python bench.py --dist --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/dist_stdout.txt 2> $OUT/dist_stderr.txt
echo done > $OUT/DONE
