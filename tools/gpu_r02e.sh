#!/bin/bash
set -u
TAG=${1:-r02e}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
timeout 600 python tools/time_pcg.py cfg5 2 > "$OUT/time_pcg_cfg5.txt" 2>&1
NSP_PRECS=2 NSP_PCG_WARM=0 NSP_GRAPH=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv \
      --log-file "$OUT/launches_pcg_cfg5.csv" python tools/time_pcg.py cfg5 1 > "$OUT/ncu_pcg_cfg5.log" 2>&1
