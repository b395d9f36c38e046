#!/bin/bash
set -u
TAG=${1:-r02p}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
NSP_SYMM_PERSIST=1 timeout 1200 python -m pytest tests/test_gpu_apply.py tests/test_gpu_edge.py tests/test_gpu_bcg.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -q -m gpu -rA -p no:cacheprovider > "$OUT/pytest_persist.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_persist.log"
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -m gpu -rA -p no:cacheprovider > "$OUT/pytest_multirank.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_multirank.log"
for v in "NSP_SYMM_PERSIST=0" "NSP_SYMM_PERSIST=1"; do
  env $v timeout 300 python tools/ab_bcg.py cfg2 15 >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
  env $v timeout 600 python tools/ab_bcg.py cfg5 3 >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
  env $v timeout 600 python tools/ab_bcg.py cfg3 5 >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
