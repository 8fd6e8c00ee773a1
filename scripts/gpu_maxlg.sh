#!/bin/bash
OUT=gpurun_out/maxlg
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_jacobi.py tests/test_gpu_dist.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for m in 5 6 7 8; do for cfg in powerlaw_8M spe10; do
  echo "== maxlg $m $cfg" >> $OUT/bench.jsonl
  HEC_TAIL_MAXLG=$m timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 200 --warmup 20 >> $OUT/bench.jsonl 2>> $OUT/bench.err
done; done
