#!/bin/bash
# BiCGSTAB count / trajectory on the power-law test matrix under SpMV knobs
OUT=gpurun_out/${1:-bicg}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python scripts/bicg_traj.py > $OUT/traj_default.json 2>&1
HEC_TAIL_MAXLG=5 python scripts/bicg_traj.py > $OUT/traj_maxlg5.json 2>&1
echo done > $OUT/DONE
