#!/bin/bash
# Tail super-block size sweep (rows regrouped within super-blocks: locality of a warp's rows vs padding).
set -u
OUT=gpurun_out/${1:-tsp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for sup in 256 512 1024 2048 4096 16384; do
  for cfg in powerlaw_8M powerlaw_8M_dsorted; do
    HEC_TAIL_SUPER=$sup timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_${cfg}_s$sup.json 2>> $OUT/err.log
  done
  HEC_TAIL_SUPER=$sup timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:"tail" -c 2 --csv --log-file $OUT/l_s$sup.csv \
     python bench.py --config powerlaw_8M --profile --steps 2 --warmup 3 > /dev/null 2>&1
done
echo done > $OUT/DONE
