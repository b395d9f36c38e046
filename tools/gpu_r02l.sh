#!/bin/bash
set -u
TAG=${1:-r02l}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
NSP_PANEL_HALF=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k panel -p no:cacheprovider > "$OUT/pytest_half.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_half.log"
for v in "NSP_PANEL_HALF=0" "NSP_PANEL_HALF=1"; do
  env $v timeout 300 python tools/ab_bcg.py cfg2 15 >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
  env $v timeout 600 python tools/ab_bcg.py cfg5 3 >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench exit $?" >> "$OUT/bench.err"
