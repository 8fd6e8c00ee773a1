#!/bin/bash
# x-ring tail schedule: parity tests, then power-law step time and per-launch ncu (ring on / off),
# for a few consumer-warp counts (HEC_RING_NW) and ring super-block sizes.
set -u
OUT=gpurun_out/${1:-ring}
NWS=${2:-16}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ring.py -x -q -p no:cacheprovider > $OUT/pytest_ring.log 2>&1; echo "rc=$?" >> $OUT/pytest_ring.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_$name.json 2>> $OUT/err.log
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:"tail|ell" -c 6 --csv --log-file $OUT/l_$name.csv \
     python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
}
run plain HEC_TAIL_RING=0
for NW in $NWS; do
  HEC_NVCC_EXTRA="-DHEC_RING_NW=$NW" python paper_1606_00545_b200/_build.py --force > $OUT/build_nw$NW.log 2>&1
  for SB in 1024 512; do
    run ring_nw${NW}_sb$SB HEC_TAIL_RING=1 HEC_TAIL_SUPER=$SB
  done
done
echo done > $OUT/DONE
