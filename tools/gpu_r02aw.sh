#!/bin/bash
# A/B: W^T slice loads trimmed to the slices that meet a product (dbg 0) vs all 7 (dbg 64); the two-CTA
# cluster variant now with the zero-slice skip
set -u
OUT=gpurun_out/${1:-r02aw}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py -q -m gpu -x > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for rep in 1 2; do
for d in 0 64; do echo "dbg $d" >> $OUT/time.txt; NSP_OZ_DBG=$d timeout 600 python tools/one_apply.py cfg5 128 0 10 >> $OUT/time.txt 2>&1; NSP_OZ_DBG=$d timeout 300 python tools/one_apply.py cfg3 64 0 20 >> $OUT/time.txt 2>&1; done
echo "cluster" >> $OUT/time.txt; NSP_OZ_CLUSTER=1 timeout 600 python tools/one_apply.py cfg5 128 0 10 >> $OUT/time.txt 2>&1
done
