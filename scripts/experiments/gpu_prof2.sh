#!/bin/bash
# Round 2 profiles: ncu --set full of the tail kernel and the ELL kernel on power-law 2^23, the ELL kernel on
# 256^3, launch lists; the cold-launch floor.
set -u
OUT=gpurun_out/${1:-pf}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python scripts/launch_floor.py > $OUT/launch_floor.json 2>> $OUT/err.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 3 -c 1 -o $OUT/prof_tail_powerlaw_8M \
  python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ell_kernel -s 3 -c 1 -o $OUT/prof_ell_powerlaw_8M \
  python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 >> $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ell_kernel -s 5 -c 1 -o $OUT/prof_ell_poisson3d_256 \
  python bench.py --profile --steps 8 --warmup 3 >> $OUT/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_poisson3d_256.csv \
  python bench.py --profile --steps 20 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_powerlaw_8M.csv \
  python bench.py --config powerlaw_8M --profile --steps 10 --warmup 3 > /dev/null 2>&1
echo done > $OUT/DONE
