#!/bin/bash
# INT8 a2+a3 v2 (fast epilogue, parallel slicer) + L22 released: tests, cfg2 timing + launch list, cfg5 bench
set -u
OUT=gpurun_out/${1:-r02u}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py tests/test_gpu_pcg.py -q -m gpu -x -s > $OUT/pytest_oz.log 2>&1; echo "exit $?" >> $OUT/pytest_oz.log
for ak in 2 3; do timeout 300 python tools/one_apply.py cfg2 128 $ak 20 >> $OUT/time.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/one_apply.py cfg2 128 3 3 > $OUT/ncu1.log 2>&1
NSP_VERBOSE=1 timeout 900 python bench.py --no-secondary --no-cpu-baseline --steps 3 --warmup 3 > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
