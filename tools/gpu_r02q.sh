#!/bin/bash
set -u
TAG=${1:-r02q}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke exit $?" >> "$OUT/smoke.log"
timeout 2400 python -m pytest tests -q -m gpu -rA -s -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench exit $?" >> "$OUT/bench.err"
timeout 900 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "ref exit $?" >> "$OUT/bench_ref.err"
