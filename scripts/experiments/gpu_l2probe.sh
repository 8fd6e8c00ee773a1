#!/bin/bash
OUT=gpurun_out/l2probe
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file $OUT/ncu.csv python scripts/l2_probe.py 20 21 22 23 > $OUT/probe.log 2>&1
