#!/bin/bash
set -u
TAG=${1:-r02n}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
./tools/bench_eig > "$OUT/bench_eig.txt" 2>&1; EIG_GRADED=1 ./tools/bench_eig >> "$OUT/bench_eig.txt" 2>&1
NSP_NYS_TRACE=1 timeout 200 python tools/time_nys.py cfg2 3 > "$OUT/nys_trace.txt" 2>&1
timeout 1200 python -m pytest tests/test_gpu_nystrom.py tests/test_gpu_bcg.py tests/test_gpu_kernels.py -q -m gpu -rA -p no:cacheprovider > "$OUT/pytest.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest.log"
NSP_PANEL_HALF=2 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k panel -p no:cacheprovider > "$OUT/pytest_half2.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_half2.log"
for v in "NSP_PANEL_HALF=0" "NSP_PANEL_HALF=1" "NSP_PANEL_HALF=2"; do
  env $v timeout 300 python tools/ab_bcg.py cfg2 15 >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
  env $v timeout 600 python tools/ab_bcg.py cfg5 3 >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
done
