#!/bin/bash
# Round-2 first GPU call: smoke, all GPU tests (no -x: every failure is reported), the dup-column
# diagnostic, the default bench line (cfg5 headline + cfg2 secondary) and the reference arm.
set -u
TAG=${1:-r02a}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"; grep -m1 "model name" /proc/cpuinfo >> "$OUT/nproc.txt"; free -g >> "$OUT/nproc.txt"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke exit $?" >> "$OUT/smoke.log"
timeout 600 python tools/diag_dup.py > "$OUT/diag_dup.log" 2>&1; echo "diag exit $?" >> "$OUT/diag_dup.log"
timeout 1800 python -m pytest tests -q -m gpu -rA -s -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench exit $?" >> "$OUT/bench.err"
timeout 600 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "ref exit $?" >> "$OUT/bench_ref.err"
