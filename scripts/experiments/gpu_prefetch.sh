#!/bin/bash
# L2 bulk prefetch (UBLKPF) of the tail's later load batches and of the ELL kernel's second-phase slots:
# power-law step time + per-launch ncu for each on/off combination; parity tests on the default build.
set -u
OUT=gpurun_out/${1:-pf}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
run() {  # name, env...
  local name=$1; shift
  for cfg in powerlaw_8M powerlaw_8M_dsorted; do
    env "$@" timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_${name}_$cfg.json 2>> $OUT/err.log
  done
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:"tail|ell" -c 6 --csv --log-file $OUT/l_${name}_powerlaw_8M.csv \
     python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
}
for V in "1 1" "0 0" "1 0" "0 1"; do
  set -- $V
  HEC_NVCC_EXTRA="-DHEC_TAIL_PREFETCH=$1 -DHEC_ELL_PREFETCH=$2" python paper_1606_00545_b200/_build.py --force > $OUT/build_$1_$2.log 2>&1
  run t$1_e$2
done
echo done > $OUT/DONE
