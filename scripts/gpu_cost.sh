#!/bin/bash
# CONTIG_COST vs CONTIG_NNZ: one-GPU compute-only projection on the power-law matrices
set -u
OUT=gpurun_out/${1:-cost}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -q > $OUT/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_dist.log
timeout 1800 python scripts/rank_emulation.py powerlaw_8M_dsorted powerlaw_8M --kind cost > $OUT/rank_emulation_cost.jsonl 2>> $OUT/err.log
echo done > $OUT/DONE
