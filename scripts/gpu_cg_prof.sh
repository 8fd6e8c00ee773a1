#!/bin/bash
OUT=gpurun_out/cg_prof
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python bench.py --solver cg --steps 100 --warmup 5 --no-cpu-baseline > $OUT/cg.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/ncu_cg.csv python bench.py --solver cg --steps 6 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
