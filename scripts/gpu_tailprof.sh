#!/bin/bash
# ncu --set full of the tail kernel (power-law) with source mapping
OUT=gpurun_out/${1:-tailprof}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 3 -c 1 -o $OUT/prof_tail \
  python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > $OUT/ncu.log 2>&1
echo done > $OUT/DONE
