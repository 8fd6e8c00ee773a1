#!/bin/bash
OUT=gpurun_out/quick3
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for cfg in poisson3d_256 poisson2d_64 spe10 powerlaw_8M; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 100 --warmup 10 >> $OUT/bench.jsonl 2>> $OUT/bench.err
done
timeout 900 python -m pytest tests/test_gpu_p2p.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
