#!/bin/bash
# Tail descriptors in reverse order (HEC_TAIL_REVERSE=1): the first tail CTAs reuse the x band / y lines
# the ELL kernel's last CTAs left in L2.  Step times, per-launch ncu, parity.
set -u
OUT=gpurun_out/${1:-rev}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
HEC_TAIL_REVERSE=1 timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for r in 0 1 0 1; do
  for cfg in powerlaw_8M powerlaw_8M_dsorted; do
    HEC_TAIL_REVERSE=$r timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_r${r}_$cfg.jsonl 2>> $OUT/err.log
  done
done
for r in 0 1; do
  for cfg in powerlaw_8M powerlaw_8M_dsorted; do
    HEC_TAIL_REVERSE=$r timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tail|ell" -c 6 --csv --log-file $OUT/l_r${r}_$cfg.csv \
      python bench.py --config $cfg --profile --steps 3 --warmup 3 > /dev/null 2>&1
  done
done
echo done > $OUT/DONE
