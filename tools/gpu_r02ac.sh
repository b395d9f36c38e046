#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02ac}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 120 python tools/one_apply.py cfg2 128 0 10 >> $OUT/time.txt 2>&1; echo "exit $?" >> $OUT/time.txt
timeout 600 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py -q -m gpu -x -s > $OUT/pytest_oz.log 2>&1; echo "exit $?" >> $OUT/pytest_oz.log
for kv in 1 2; do echo "kernel $kv" >> $OUT/time.txt; NSP_OZ_KERNEL=$kv timeout 600 python tools/one_apply.py cfg5 128 0 10 >> $OUT/time.txt 2>&1; NSP_OZ_KERNEL=$kv timeout 300 python tools/one_apply.py cfg2 128 0 20 >> $OUT/time.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg5.csv python tools/one_apply.py cfg5 128 0 2 > $OUT/ncu_l5.log 2>&1
