#!/bin/bash
# ELL index compression, quick: parity tests + 256^3 / 150^3 / SPE10 bench with and without.
set -u
OUT=gpurun_out/${1:-idx16b}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_idx16.py -q -p no:cacheprovider > $OUT/pytest_idx16.log 2>&1; echo "rc=$?" >> $OUT/pytest_idx16.log
for cfg in poisson3d_256 poisson3d_150 spe10; do
  for f in 1 0; do
    HEC_IDX16=$f timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_${cfg}_idx$f.json 2>> $OUT/err.log
  done
done
echo done > $OUT/DONE
