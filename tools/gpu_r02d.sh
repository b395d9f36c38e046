#!/bin/bash
set -u
TAG=${1:-r02d}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
timeout 300 python tools/time_nys.py cfg2 4 > "$OUT/time_nys.txt" 2>&1
NSP_FUSED_SXS=0 timeout 300 python tools/time_nys.py cfg2 4 > "$OUT/time_nys_sxs0.txt" 2>&1
NSP_GRAPH=1 timeout 300 python tools/time_nys.py cfg2 3 > "$OUT/time_nys_graph1.txt" 2>&1
SHORT2="python bench.py --config cfg2 --steps 1 --warmup 3 --apply-reps 2 --no-cpu-baseline --no-secondary --no-nystrom"
NSP_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
      --log-file "$OUT/launches_cfg2.csv" $SHORT2 > "$OUT/ncu_launches_cfg2.log" 2>&1
timeout 300 python tools/time_pcg.py cfg2 5 > "$OUT/time_pcg.txt" 2>&1
