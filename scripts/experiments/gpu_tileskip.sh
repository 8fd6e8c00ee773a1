#!/bin/bash
# ELL second-phase slot skipping (tile_w): parity, degree-sorted and power-law lines with it on/off;
# and the power-law line's dependence on steps/warm-up (100/10 vs 200/20) and on the post-timing passes.
set -u
OUT=gpurun_out/${1:-ts}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tileskip.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for f in 1 0; do
  HEC_TILE_SKIP=$f timeout 600 python bench.py --config powerlaw_8M_dsorted --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_dsorted_skip$f.jsonl 2>> $OUT/err.log
  HEC_TILE_SKIP=$f timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tail|ell" -c 6 --csv --log-file $OUT/l_dsorted_skip$f.csv \
      python bench.py --config powerlaw_8M_dsorted --profile --steps 3 --warmup 3 > /dev/null 2>&1
done
for f in 1 0; do
  HEC_TILE_SKIP=$f timeout 600 python bench.py --config powerlaw_8M_dsorted --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_dsorted_skip$f.jsonl 2>> $OUT/err.log
done
for i in 1 2; do
  timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_pl_100.jsonl 2>> $OUT/err.log
  timeout 600 python bench.py --config powerlaw_8M --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-ncu --no-anchor >> $OUT/b_pl_200.jsonl 2>> $OUT/err.log
  timeout 900 python bench.py --config powerlaw_8M --no-cpu-baseline --no-anchor >> $OUT/b_pl_full.jsonl 2>> $OUT/err.log
done
echo done > $OUT/DONE
