#!/bin/bash
# SM-local persistent tail schedule: parity, power-law timing on/off, launch list, ncu capture.
set -u
OUT=gpurun_out/${1:-ts}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for sm in 1 0; do
  for cfg in powerlaw_8M powerlaw_8M_dsorted; do
    HEC_TAIL_SM=$sm timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-ncu --no-anchor > $OUT/b_${cfg}_sm$sm.json 2>> $OUT/err.log
  done
  HEC_TAIL_SM=$sm timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:"tail" -c 3 --csv --log-file $OUT/l_sm$sm.csv \
     python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_sm -s 2 -c 1 -o $OUT/prof_tail_sm \
  python bench.py --config powerlaw_8M --profile --steps 3 --warmup 3 > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
