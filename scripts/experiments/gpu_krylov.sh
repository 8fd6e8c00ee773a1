#!/bin/bash
OUT=gpurun_out/krylov
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_p2p.py tests/test_gpu_dist.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python scripts/cg_probe.py > $OUT/probe.log 2>&1
timeout 600 python bench.py --solver cg --steps 100 --warmup 5 > $OUT/cg.json 2>> $OUT/bench.err
timeout 600 python bench.py --solver bicgstab --steps 100 --warmup 5 > $OUT/bicgstab.json 2>> $OUT/bench.err
