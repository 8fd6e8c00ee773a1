#!/bin/bash
# Per-step time series of the power-law SpMV under a few settings (is the slow-step mode periodic, thermal,
# or tied to the programmatic-dependent launch / the tail order?)
set -u
OUT=gpurun_out/${1:-ser}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python scripts/step_series.py powerlaw_8M 400 > $OUT/s_default.json 2>> $OUT/err.log
python scripts/step_series.py powerlaw_8M 400 HEC_PDL=0 > $OUT/s_nopdl.json 2>> $OUT/err.log
python scripts/step_series.py powerlaw_8M 400 HEC_TAIL_REVERSE=0 > $OUT/s_norev.json 2>> $OUT/err.log
python scripts/step_series.py poisson3d_256 400 > $OUT/s_256.json 2>> $OUT/err.log
python scripts/step_series.py powerlaw_8M_dsorted 400 > $OUT/s_dsorted.json 2>> $OUT/err.log
echo done > $OUT/DONE
