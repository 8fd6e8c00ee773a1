#!/bin/bash
# Grouped distributed sub-matrices: parity (tile-skip/grouping tests, distributed + full-size suites)
# and the --dist N = 1 power-law line with and without grouping.
set -u
OUT=gpurun_out/${1:-dg}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_tileskip.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py tests/test_gpu_p2p.py tests/test_gpu_krylov.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do
  for f in 1 0; do
    HEC_ELL_GROUP=$f timeout 600 python bench.py --dist --config powerlaw_8M --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_dist_g$f.jsonl 2>> $OUT/err.log
  done
done
timeout 600 python scripts/rank_emulation.py powerlaw_8M > $OUT/rank_emulation.jsonl 2>> $OUT/err.log
echo done > $OUT/DONE
