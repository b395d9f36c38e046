#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02ae}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
NSP_PRECS=2 timeout 300 python tools/time_pcg.py cfg2 7 > $OUT/time_pcg_cfg2.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_pcg_cfg2.csv python tools/one_pcg.py cfg2 30 > $OUT/ncu_pcg.log 2>&1
