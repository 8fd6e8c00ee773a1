#!/bin/bash
# Round 2 check: full GPU suite, smoke, tail-heavy and small bench lines, Jacobi on the tail, a last epl point.
set -u
OUT=gpurun_out/${1:-r2c}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for cfg in powerlaw_8M powerlaw_8M_dsorted spe10 poisson3d_128 poisson2d_64; do
  timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_$cfg.json 2>> $OUT/bench.err
done
HEC_FUSE_TAIL=0 timeout 600 python bench.py --config spe10 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_spe10_nofuse.json 2>> $OUT/bench.err
HEC_TAIL_EPL=64 timeout 600 python bench.py --config powerlaw_8M --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_powerlaw_8M_epl64.json 2>> $OUT/bench.err
timeout 600 python bench.py --jacobi 0.8 --config powerlaw_8M --steps 50 --warmup 5 > $OUT/jacobi_powerlaw.json 2>> $OUT/bench.err
timeout 600 python bench.py --dist --config powerlaw_8M --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_dist_n1_powerlaw.json 2>> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ell_kernel|tail" -c 8 --csv --log-file $OUT/launches_spe10.csv \
  python bench.py --config spe10 --profile --steps 3 --warmup 3 > /dev/null 2>&1
echo done > $OUT/DONE
