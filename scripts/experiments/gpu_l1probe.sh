#!/bin/bash
# Is the power-law tail bound by L1 sector throughput?  Drop the value stream (EXPERIMENT build, wrong
# results) and see whether the time falls with the sector count; also the TMA ELL variant on the power-law.
set -u
OUT=gpurun_out/${1:-l1p}
mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed"
python paper_1606_00545_b200/_build.py --force > $OUT/build0.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"tail|ell" -c 4 --csv --log-file $OUT/l_base.csv python bench.py --config powerlaw_8M --profile --steps 2 --warmup 2 > /dev/null 2>&1
HEC_ELL_KERNEL=tma timeout 600 ncu --metrics $M --clock-control none -k regex:"tail|ell" -c 4 --csv --log-file $OUT/l_ell_tma.csv python bench.py --config powerlaw_8M --profile --steps 2 --warmup 2 > /dev/null 2>&1
HEC_ELL_KERNEL=tma timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-anchor --no-ncu > $OUT/b_ell_tma.json 2>> $OUT/err.log
HEC_NVCC_EXTRA="-DHEC_TAIL_NOVAL=1" python paper_1606_00545_b200/_build.py --force > $OUT/build1.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"tail" -c 2 --csv --log-file $OUT/l_noval.csv python bench.py --config powerlaw_8M --profile --steps 2 --warmup 2 > /dev/null 2>&1
python paper_1606_00545_b200/_build.py --force > $OUT/build2.log 2>&1
echo done > $OUT/DONE
