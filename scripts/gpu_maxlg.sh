#!/bin/bash
OUT=gpurun_out/maxlg2
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for e in 4 6 8 12; do
  echo "== epl $e" >> $OUT/bench.jsonl
  HEC_TAIL_EPL=$e timeout 600 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e --steps 200 --warmup 20 >> $OUT/bench.jsonl 2>> $OUT/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file $OUT/launches.csv python bench.py --config powerlaw_8M --profile --steps 5 --warmup 1 > /dev/null 2>&1
