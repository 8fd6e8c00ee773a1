#!/bin/bash
# Round profile: tests, smoke, bench lines (all configs + NEXT rows), reference
# arm, ncu launch lists, and one ncu --set full capture per hot kernel.
set -u
TAG=${1:-round1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2>> $OUT/bench.err
for cfg in poisson3d_128 spe10 powerlaw_8M poisson3d_150 poisson2d_64 powerlaw_8M_dsorted; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > $OUT/bench_$cfg.json 2>> $OUT/bench.err
done
timeout 600 python bench.py --dist --steps 100 --warmup 5 --no-cpu-baseline > $OUT/bench_dist_n1.json 2>> $OUT/bench.err
for s in cg bicgstab; do timeout 600 python bench.py --solver $s --steps 100 --warmup 5 > $OUT/solver_$s.json 2>> $OUT/bench.err; done
for cfg in poisson3d_256 spe10 powerlaw_8M; do timeout 600 python bench.py --jacobi 0.8 --config $cfg --steps 100 --warmup 5 >> $OUT/jacobi.jsonl 2>> $OUT/bench.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_poisson3d_256.csv \
  python bench.py --profile --steps 20 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/launches_powerlaw_8M.csv \
  python bench.py --config powerlaw_8M --profile --steps 10 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $OUT/launches_p2p_local_256_p8.csv \
  python scripts/p2p_local_probe.py 8 > $OUT/p2p_local.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ell_kernel -s 5 -c 1 -o $OUT/prof_ell_poisson3d_256 \
  python bench.py --profile --steps 8 --warmup 3 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 3 -c 1 -o $OUT/prof_tail_powerlaw_8M \
  python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 >> $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ell_kernel -s 3 -c 1 -o $OUT/prof_ell_powerlaw_8M \
  python bench.py --config powerlaw_8M --profile --steps 5 --warmup 3 >> $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
