#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02ao}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 120 python tools/one_apply.py cfg2 128 0 5 >> $OUT/time.txt 2>&1; echo "exit $?" >> $OUT/time.txt
timeout 600 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py -q -m gpu -x > $OUT/pytest_oz.log 2>&1; echo "exit $?" >> $OUT/pytest_oz.log
for d in 0 16; do echo "dbg $d" >> $OUT/time.txt; NSP_OZ_DBG=$d timeout 600 python tools/one_apply.py cfg5 128 0 10 >> $OUT/time.txt 2>&1; NSP_OZ_DBG=$d timeout 300 python tools/one_apply.py cfg2 128 0 20 >> $OUT/time.txt 2>&1;
NSP_OZ_DBG=$d timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:oz_symm -s 1 -c 1 python tools/one_apply.py cfg5 128 0 1 >> $OUT/time.txt 2>&1; done
