#!/bin/bash
set -u
TAG=${1:-r02j}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
timeout 600 python tools/trace_bcg.py cfg5 > "$OUT/trace_cfg5.txt" 2>&1
timeout 300 python tools/trace_bcg.py cfg2 > "$OUT/trace_cfg2.txt" 2>&1
for v in "NSP_XFORK=1" "NSP_XFORK=0" "NSP_APPLY_FIRST=1"; do
  env $v timeout 600 python tools/ab_bcg.py cfg5 3 >> "$OUT/ab_cfg5.jsonl" 2>> "$OUT/ab.err"
done
