#!/bin/bash
set -u
TAG=${1:-r02i}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
timeout 1200 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_nystrom.py tests/test_gpu_edge.py tests/test_gpu_multirank.py -q -m gpu -rA -p no:cacheprovider > "$OUT/pytest.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest.log"
NSP_PRECS=2,1 NSP_PCG_WARM=1 timeout 600 python tools/time_pcg.py cfg5 2 > "$OUT/time_pcg_cfg5.txt" 2>&1
NSP_PRECS=2,1 timeout 600 python tools/time_pcg.py cfg2 5 > "$OUT/time_pcg_cfg2.txt" 2>&1
timeout 300 python tools/ab_bcg.py cfg2 15 --analog > "$OUT/ab_cfg2.jsonl" 2>&1
