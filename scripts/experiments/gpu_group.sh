#!/bin/bash
# ELL rows grouped by length (4096-row windows) + second-phase slot skipping: full GPU suite on the
# default build, then A/B on one box (grouped+skip vs neither), alternating, and per-launch ncu.
set -u
OUT=gpurun_out/${1:-grp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for i in 1 2; do
  for v in on off; do
    if [ $v = on ]; then E=""; else E="HEC_ELL_GROUP=0 HEC_TILE_SKIP=0"; fi
    for cfg in powerlaw_8M powerlaw_8M_dsorted; do
      env $E timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_${v}_$cfg.jsonl 2>> $OUT/err.log
    done
  done
done
for v in on off; do
  if [ $v = on ]; then E=""; else E="HEC_ELL_GROUP=0 HEC_TILE_SKIP=0"; fi
  env $E timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tail|ell" -c 6 --csv --log-file $OUT/l_${v}_powerlaw_8M.csv \
      python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
done
echo done > $OUT/DONE
