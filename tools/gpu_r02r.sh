#!/bin/bash
set -u
TAG=${1:-r02r}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
s=$(date +%s); timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench exit $? wall $(( $(date +%s) - s )) s" >> "$OUT/bench.err"
s=$(date +%s); timeout 900 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "ref exit $? wall $(( $(date +%s) - s )) s" >> "$OUT/bench_ref.err"
