#!/bin/bash
# Grouping window size (HEC_GROUP_ROWS 512 / 1024 / 4096) vs no grouping, one box, alternating; per-launch ncu.
set -u
OUT=gpurun_out/${1:-grp2}
mkdir -p $OUT
for G in 512 1024 4096; do
  HEC_NVCC_EXTRA="-DHEC_GROUP_ROWS=$G" python paper_1606_00545_b200/_build.py --force > $OUT/build_$G.log 2>&1
  for i in 1 2; do
    timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_g$G.jsonl 2>> $OUT/err.log
    HEC_ELL_GROUP=0 timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_nogroup.jsonl 2>> $OUT/err.log
  done
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:"ell" -c 3 --csv --log-file $OUT/l_g$G.csv \
      python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
done
HEC_ELL_GROUP=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:"ell" -c 3 --csv --log-file $OUT/l_nogroup.csv \
    python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
python paper_1606_00545_b200/_build.py --force > $OUT/build_default.log 2>&1
echo done > $OUT/DONE
