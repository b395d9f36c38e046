#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02ab}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 300 python tools/one_apply.py cfg2 128 0 10 >> $OUT/time.txt 2>&1; echo "exit $?" >> $OUT/time.txt
timeout 600 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py -q -m gpu -x -s > $OUT/pytest_oz.log 2>&1; echo "exit $?" >> $OUT/pytest_oz.log
for cl in 0 1; do echo "cluster $cl" >> $OUT/time.txt; NSP_OZ_CLUSTER=$cl timeout 600 python tools/one_apply.py cfg5 128 0 10 >> $OUT/time.txt 2>&1; NSP_OZ_CLUSTER=$cl timeout 300 python tools/one_apply.py cfg2 128 0 20 >> $OUT/time.txt 2>&1; done
