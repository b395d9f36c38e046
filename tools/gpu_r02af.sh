#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02af}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py -q -m gpu -x -s > $OUT/pytest_oz.log 2>&1; echo "exit $?" >> $OUT/pytest_oz.log
for c in cfg5 cfg2; do timeout 600 python tools/one_apply.py $c 128 0 10 >> $OUT/time.txt 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_symm -s 1 -c 1 -o $OUT/oz_symm_cfg5 python tools/one_apply.py cfg5 128 0 1 > $OUT/ncu_cfg5.log 2>&1
