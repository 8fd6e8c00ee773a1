#!/bin/bash
# Tail kernels (warp-chunk layout; plain and x-window): GPU suite, power-law timing with the window on/off,
# ncu launch list and one full capture of each tail kernel.
set -u
OUT=gpurun_out/${1:-tw}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for w in 1 0; do
  HEC_TAIL_WIN=$w timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_pl_win$w.json 2>> $OUT/bench.err
  HEC_TAIL_WIN=$w timeout 600 python bench.py --config powerlaw_8M_dsorted --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_pld_win$w.json 2>> $OUT/bench.err
done
timeout 600 python bench.py --config spe10 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_spe10.json 2>> $OUT/bench.err
for w in 1 0; do
HEC_TAIL_WIN=$w timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ell_kernel|tail" -c 6 --csv --log-file $OUT/launches_pl_win$w.csv \
  python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_win -s 3 -c 1 -o $OUT/prof_tailwin \
  python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > $OUT/ncu_full.log 2>&1
HEC_TAIL_WIN=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 3 -c 1 -o $OUT/prof_tail \
  python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 >> $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
