#!/bin/bash
set -u
TAG=${1:-r02k}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
for v in default nw8 gns4 g1gns4; do
  if [ $v = default ]; then L=""; else L="NSP_LIB=tools/variants/$v/libnsp.so"; fi
  echo "$v" >> "$OUT/ab.jsonl"
  env $L timeout 300 python tools/ab_bcg.py cfg2 15 >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
  env $L timeout 600 python tools/ab_bcg.py cfg5 3 >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
