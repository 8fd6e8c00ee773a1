#!/bin/bash
# Degree-sorted power-law variant (SURVEY §8(d) secondary row): parity, N=1
# bench line, and the one-GPU compute-only projection of P = 1..8 parts
set -u
OUT=gpurun_out/${1:-ranks}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spmv.py -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --config powerlaw_8M_dsorted --no-cpu-baseline > $OUT/bench_powerlaw_8M_dsorted.json 2>> $OUT/err.log
timeout 1800 python scripts/rank_emulation.py poisson3d_256 powerlaw_8M powerlaw_8M_dsorted > $OUT/rank_emulation.jsonl 2>> $OUT/err.log
echo done > $OUT/DONE
