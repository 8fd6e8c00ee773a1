#!/bin/bash
# Refresh of the numbers that depend on the tail kernel: rank projection and the Table-3 analog
set -u
OUT=gpurun_out/${1:-refresh2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python scripts/rank_emulation.py poisson3d_256 powerlaw_8M powerlaw_8M_dsorted > $OUT/rank_emulation.jsonl 2>> $OUT/err.log
timeout 1800 python bench.py --formats all > $OUT/formats.jsonl 2>> $OUT/err.log
echo done > $OUT/DONE
