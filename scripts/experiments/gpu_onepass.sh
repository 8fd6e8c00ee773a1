#!/bin/bash
# One-pass HEC kernel: parity tests, then power-law step time + per-launch ncu over tile sizes / grids.
set -u
OUT=gpurun_out/${1:-onepass}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_onepass.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_$name.json 2>> $OUT/err.log
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:"tail|ell|fused" -c 6 --csv --log-file $OUT/l_$name.csv \
     python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
}
run plain HEC_FUSED=0
for R in 2048 1024 512 4096; do
  run r$R HEC_FUSED=1 HEC_FUSED_ROWS=$R
done
run r2048_g5 HEC_FUSED=1 HEC_FUSED_ROWS=2048 HEC_FUSED_GRID=5
run r1024_g6 HEC_FUSED=1 HEC_FUSED_ROWS=1024 HEC_FUSED_GRID=6
HEC_FUSED=1 timeout 600 python bench.py --config powerlaw_8M_dsorted --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_dsorted_r2048.json 2>> $OUT/err.log
timeout 600 python bench.py --config powerlaw_8M_dsorted --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_dsorted_plain.json 2>> $OUT/err.log
echo done > $OUT/DONE
