#!/bin/bash
# Round 2: GPU suite + smoke + SPE10 fused / two-kernel bench lines + launch list.
set -u
OUT=gpurun_out/${1:-r2d}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --config spe10 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_spe10.json 2>> $OUT/bench.err
HEC_FUSE_TAIL=0 timeout 600 python bench.py --config spe10 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_spe10_nofuse.json 2>> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ell_kernel|tail" -c 8 --csv --log-file $OUT/launches_spe10.csv \
  python bench.py --config spe10 --profile --steps 3 --warmup 3 > /dev/null 2>&1
echo done > $OUT/DONE
