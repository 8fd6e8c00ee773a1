#!/bin/bash
set -u
TAG=${1:-r14}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for cfg in poisson3d_256 poisson3d_128 spe10; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline > $OUT/b_$cfg.json 2>> $OUT/err.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --dist --steps 50 --warmup 5 > $OUT/b_dist1_poisson3d_256.json 2>> $OUT/err.log
timeout 600 python bench.py --dist --config powerlaw_8M --steps 20 --warmup 3 > $OUT/b_dist1_powerlaw.json 2>> $OUT/err.log
echo done > $OUT/DONE
