#!/bin/bash
# Tail kernel variants (compile-time HEC_TAIL_V / HEC_TAIL_UNROLL, runtime HEC_TAIL_EPL / HEC_TAIL_WIN):
# power-law step time + ncu per-launch time and DRAM bytes of the tail kernel.
set -u
OUT=gpurun_out/${1:-tv}
mkdir -p $OUT
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_$name.json 2>> $OUT/err.log
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"tail" -c 3 --csv --log-file $OUT/l_$name.csv \
     python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
}
for V in "0 2" "0 4" "3 2" "4 2"; do
  set -- $V
  HEC_NVCC_EXTRA="-DHEC_TAIL_V=$1 -DHEC_TAIL_UNROLL=$2" python paper_1606_00545_b200/_build.py --force > $OUT/build_v$1_u$2.log 2>&1
  run v$1_u$2_win0 HEC_TAIL_WIN=0
  run v$1_u$2_win1 HEC_TAIL_WIN=1
  if [ "$1" = "0" ] && [ "$2" = "2" ]; then
    run v0_u2_epl16_win0 HEC_TAIL_WIN=0 HEC_TAIL_EPL=16
    run v0_u2_epl4_win0 HEC_TAIL_WIN=0 HEC_TAIL_EPL=4
    run v0_u2_epl16_win1 HEC_TAIL_WIN=1 HEC_TAIL_EPL=16
  fi
done
python paper_1606_00545_b200/_build.py --force > $OUT/build_final.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tailwin.py tests/test_gpu_fullsize.py tests/test_gpu_spmv.py tests/test_gpu_jacobi.py -q -p no:cacheprovider -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
echo done > $OUT/DONE
