#!/bin/bash
set -u
TAG=${1:-r02m}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
NSP_NYS_TRACE=1 timeout 200 python tools/time_nys.py cfg2 2 > "$OUT/nys_trace.txt" 2>&1
timeout 1200 python -m pytest tests/test_gpu_nystrom.py tests/test_gpu_bcg.py tests/test_gpu_pcg.py tests/test_gpu_edge.py -q -m gpu -rA -p no:cacheprovider > "$OUT/pytest.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest.log"
for v in "NSP_CHEB_SELL=0" "NSP_CHEB_SELL=1"; do
  echo "$v" >> "$OUT/time_pcg_cfg5.txt"
  env $v NSP_PRECS=2,1 NSP_PCG_WARM=1 timeout 600 python tools/time_pcg.py cfg5 2 >> "$OUT/time_pcg_cfg5.txt" 2>&1
done
NSP_NYS_TRACE=1 timeout 600 python tools/time_nys.py cfg5 2 > "$OUT/nys_trace_cfg5.txt" 2>&1
