#!/bin/bash
set -u
TAG=${1:-r02o}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke exit $?" >> "$OUT/smoke.log"
EIG_FILE=tools/C_cfg2.bin ./tools/bench_eig > "$OUT/eigC.txt" 2>&1
NSP_NYS_TRACE=1 timeout 200 python tools/time_nys.py cfg2 3 > "$OUT/nys_trace.txt" 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rA -s -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench exit $?" >> "$OUT/bench.err"
