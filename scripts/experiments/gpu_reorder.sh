#!/bin/bash
set -u
OUT=gpurun_out/reorder
mkdir -p $OUT
timeout 600 python bench.py --config poisson3d_128 --no-cpu-baseline --no-e2e --scramble 1 > $OUT/p128_scr.json 2>> $OUT/err.log
timeout 600 python bench.py --config poisson3d_128 --no-cpu-baseline --no-e2e --scramble 1 --reorder rcm > $OUT/p128_scr_rcm.json 2>> $OUT/err.log
timeout 900 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e --reorder rcm > $OUT/pl_rcm.json 2>> $OUT/err.log
timeout 900 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e --scramble 2 > $OUT/pl_scr.json 2>> $OUT/err.log
timeout 900 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e --scramble 2 --reorder rcm > $OUT/pl_scr_rcm.json 2>> $OUT/err.log
echo done > $OUT/DONE
