#!/bin/bash
# ELL index compression: parity tests, full GPU suite, bench lines with and without (HEC_IDX16=0),
# per-launch ncu of the 256^3 ELL kernel.
set -u
OUT=gpurun_out/${1:-idx16}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_idx16.py -x -q -p no:cacheprovider > $OUT/pytest_idx16.log 2>&1; echo "rc=$?" >> $OUT/pytest_idx16.log
for cfg in poisson3d_256 poisson3d_150 poisson3d_128 spe10; do
  for f in 1 0; do
    HEC_IDX16=$f timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_${cfg}_idx$f.json 2>> $OUT/err.log
  done
done
for f in 1 0; do
  HEC_IDX16=$f timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ell" -c 6 --csv --log-file $OUT/l_poisson3d_256_idx$f.csv \
     python bench.py --profile --steps 3 --warmup 3 > /dev/null 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
