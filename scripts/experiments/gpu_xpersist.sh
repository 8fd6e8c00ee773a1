#!/bin/bash
# L2 persisting access-policy window over x (HEC_X_PERSIST=1) on the configs with scattered x gathers.
set -u
OUT=gpurun_out/${1:-xp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python -c "
import torch; p=torch.cuda.get_device_properties(0); print(p)
import ctypes
" > $OUT/props.txt 2>&1
for cfg in powerlaw_8M_dsorted powerlaw_8M poisson3d_256; do
  for f in 0 1; do
    HEC_X_PERSIST=$f timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_${cfg}_xp$f.json 2>> $OUT/err.log
    HEC_X_PERSIST=$f timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"tail|ell" -c 6 --csv --log-file $OUT/l_${cfg}_xp$f.csv \
      python bench.py --config $cfg --profile --steps 3 --warmup 3 > /dev/null 2>&1
  done
done
HEC_X_PERSIST=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k powerlaw > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
echo done > $OUT/DONE
