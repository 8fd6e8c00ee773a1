#!/bin/bash
# Tail x gathers with an L2 evict_last policy (HEC_TAIL_XHINT) A/B, two rounds each
set -u
OUT=gpurun_out/${1:-xhint}; mkdir -p $OUT
for H in 0 1 0 1; do
  HEC_NVCC_EXTRA="-DHEC_TAIL_XHINT=$H" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
  timeout 300 python bench.py --config powerlaw_8M --no-cpu-baseline --no-e2e >> $OUT/b_powerlaw_8M_h$H.jsonl 2>> $OUT/err.log
done
HEC_NVCC_EXTRA="-DHEC_TAIL_XHINT=1" python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -s 6 -c 4 --csv --log-file $OUT/launches_h1.csv \
    python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > /dev/null 2>&1
python -c "from paper_1606_00545_b200 import _build; _build.build(force=True)" >> $OUT/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -s 6 -c 4 --csv --log-file $OUT/launches_h0.csv \
    python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 > /dev/null 2>&1
echo done > $OUT/DONE
