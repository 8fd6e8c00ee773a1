#!/bin/bash
# x-ring tail schedule, round 2 of the sweep: dynamic unit claims (biggest first) and D stages in
# flight; consumer warps NW x depth D x super-block rows SB x batch B; ncu --set full of the first.
set -u
OUT=gpurun_out/${1:-ring2}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ring.py -x -q -p no:cacheprovider > $OUT/pytest_ring.log 2>&1; echo "rc=$?" >> $OUT/pytest_ring.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_$name.json 2>> $OUT/err.log
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:"tail|ell" -c 6 --csv --log-file $OUT/l_$name.csv \
     python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
}
first=1
for V in "16 3 1024 8" "16 4 512 8" "24 3 1024 8" "31 3 1024 4" "31 4 512 4" "31 3 1024 8"; do
  set -- $V
  HEC_NVCC_EXTRA="-DHEC_RING_NW=$1 -DHEC_RING_DEPTH=$2 -DHEC_RING_BATCH=$4" python paper_1606_00545_b200/_build.py --force > $OUT/build_$1_$2_$4.log 2>&1
  run nw$1_d$2_sb$3_b$4 HEC_TAIL_RING=1 HEC_TAIL_SUPER=$3
  if [ $first = 1 ]; then
    first=0
    HEC_TAIL_RING=1 HEC_TAIL_SUPER=$3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tail_ring -s 3 -c 1 -o $OUT/prof_ring \
      python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > $OUT/ncu_full.log 2>&1
  fi
done
echo done > $OUT/DONE
