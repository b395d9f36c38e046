#!/bin/bash
# INT8 tensor-core a2+a3 (reading R10): build, parity tests, cfg2 bench line, then cfg5 bench line
set -u
TAG=${1:-r02s}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
timeout 600 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py -q -m gpu -x -s > "$OUT/pytest_oz.log" 2>&1; echo "exit $?" >> "$OUT/pytest_oz.log"
NSP_VERBOSE=1 timeout 300 python bench.py --config cfg2 --no-secondary --no-cpu-baseline --steps 5 --warmup 3 > "$OUT/bench_cfg2.json" 2> "$OUT/bench_cfg2.err"
NSP_VERBOSE=1 timeout 900 python bench.py --no-secondary --no-cpu-baseline --steps 3 --warmup 3 > "$OUT/bench_cfg5.json" 2> "$OUT/bench_cfg5.err"
