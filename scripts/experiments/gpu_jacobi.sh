#!/bin/bash
# NEXT-3 Jacobi epilogue: GPU parity + sweep timing
OUT=gpurun_out/jacobi
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_jacobi.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for cfg in poisson3d_256 poisson3d_150 spe10 powerlaw_8M; do
  timeout 600 python bench.py --jacobi 0.8 --config $cfg --steps 100 --warmup 5 >> $OUT/bench_jacobi.jsonl 2>> $OUT/bench.err
done
