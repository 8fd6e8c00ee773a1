#!/bin/bash
OUT=gpurun_out/p2p
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_dist.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --dist --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_dist.json 2> $OUT/bench_dist.err
