#!/bin/bash
# Fused small tail: parity + SPE10 fused / two-kernel bench lines + launch list.
set -u
OUT=gpurun_out/${1:-fu}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_spmv.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do
timeout 600 python bench.py --config spe10 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_spe10_$i.json 2>> $OUT/bench.err
HEC_FUSE_TAIL=0 timeout 600 python bench.py --config spe10 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/bench_spe10_nofuse_$i.json 2>> $OUT/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ell_kernel|tail" -c 6 --csv --log-file $OUT/launches_spe10.csv \
  python bench.py --config spe10 --profile --steps 3 --warmup 3 > /dev/null 2>&1
HEC_FUSE_TAIL=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ell_kernel|tail" -c 6 --csv --log-file $OUT/launches_spe10_nofuse.csv \
  python bench.py --config spe10 --profile --steps 3 --warmup 3 > /dev/null 2>&1
echo done > $OUT/DONE
