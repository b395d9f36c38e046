#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02as}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py tests/test_gpu_bench_path.py -q -m gpu -x > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for d in 0 32; do echo "dbg $d" >> $OUT/time.txt; NSP_VERBOSE=1 NSP_OZ_DBG=$d timeout 600 python tools/one_apply.py cfg5 128 0 10 >> $OUT/time.txt 2>&1; NSP_VERBOSE=1 NSP_OZ_DBG=$d timeout 300 python tools/one_apply.py cfg2 128 0 20 >> $OUT/time.txt 2>&1; NSP_VERBOSE=1 NSP_OZ_DBG=$d timeout 300 python tools/one_apply.py cfg3 64 0 20 >> $OUT/time.txt 2>&1; done
