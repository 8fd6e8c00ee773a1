#!/bin/bash
# ELL x window in shared memory (HEC_ELL_WIN=1, window columns HEC_ELL_WIN_COLS): parity, then the power-law,
# degree-sorted and 256^3 steps on one box, alternating with the plain ELL; per-launch ncu.
set -u
OUT=gpurun_out/${1:-ew}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tileskip.py -q -p no:cacheprovider -k x_window > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do
  for v in "0 0" "1 6144" "1 9216" "1 12288"; do
    set -- $v
    for cfg in powerlaw_8M powerlaw_8M_dsorted; do
      HEC_ELL_WIN=$1 HEC_ELL_WIN_COLS=$2 timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_w$1_$2_$cfg.jsonl 2>> $OUT/err.log
    done
  done
done
for v in "0 0" "1 9216"; do
  set -- $v
  HEC_ELL_WIN=$1 HEC_ELL_WIN_COLS=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:"ell" -c 3 --csv --log-file $OUT/l_w$1_powerlaw_8M.csv \
      python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
  HEC_ELL_WIN=$1 HEC_ELL_WIN_COLS=$2 timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_w$1_256.jsonl 2>> $OUT/err.log
done
echo done > $OUT/DONE
