#!/bin/bash
# Small (cold, launch/ramp-bound) configs: ELL CTA size and grid cap sweep, tail order.
set -u
OUT=gpurun_out/${1:-sm}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
b() { local name=$1; shift; env "$@" timeout 300 python bench.py --config $CFG --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_${CFG}_$name.json 2>> $OUT/err.log; }
for CFG in spe10 poisson3d_128; do
  b base
  for bs in 64 256; do b blk$bs HEC_ELL_BLOCK=$bs; done
  for c in 8 10 16 20; do b cap$c HEC_ELL_CAP=$c; done
  b nofuse HEC_FUSE_TAIL=0
  b nopdl HEC_PDL=0 HEC_FUSE_TAIL=0
done
echo done > $OUT/DONE
