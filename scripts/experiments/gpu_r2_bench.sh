#!/bin/bash
# Round 2: bench lines (default, reference, --dist N=1 path, other configs).
set -u
OUT=gpurun_out/${1:-r2b}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2>> $OUT/bench.err
timeout 600 python bench.py --dist --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_dist_n1.json 2>> $OUT/bench.err
timeout 600 python bench.py --dist --config powerlaw_8M --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_dist_n1_powerlaw.json 2>> $OUT/bench.err
timeout 600 python -m pytest tests/test_gpu_krylov.py -q -p no:cacheprovider > $OUT/pytest_krylov.log 2>&1; echo "rc=$?" >> $OUT/pytest_krylov.log
echo done > $OUT/DONE
