#!/bin/bash
# Tail super-block size sweep (HEC_TAIL_SUPER) on the power-law step
set -u
OUT=gpurun_out/${1:-tailsuper}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for S in 1024 2048 4096 8192 16384 65536; do
  HEC_TAIL_SUPER=$S timeout 300 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e > $OUT/b_powerlaw_8M_s$S.json 2>> $OUT/err.log
done
HEC_TAIL_SUPER=16384 timeout 300 python bench.py --config spe10 --no-cpu-baseline --no-e2e > $OUT/b_spe10_s16384.json 2>> $OUT/err.log
echo done > $OUT/DONE
