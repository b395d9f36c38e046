#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02x}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py tests/test_gpu_bench_path.py -q -m gpu -x -s > $OUT/pytest_oz.log 2>&1; echo "exit $?" >> $OUT/pytest_oz.log
for c in cfg2 cfg5; do timeout 600 python tools/one_apply.py $c 128 0 10 >> $OUT/time.txt 2>&1; done
