#!/bin/bash
OUT=gpurun_out/e2e2
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_spmv.py -q -x -k "host" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for r in 1 0 1 0; do
  echo "== ramp $r" >> $OUT/bench.jsonl
  HEC_HOST_RAMP=$r timeout 600 python bench.py --no-cpu-baseline --steps 50 --warmup 5 >> $OUT/bench.jsonl 2>> $OUT/bench.err
done
python scripts/pcie_probe.py > $OUT/pcie.json 2>&1
