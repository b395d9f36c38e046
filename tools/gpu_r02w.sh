#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02w}; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/b tools/bench_i8mma.cu && timeout 120 /tmp/b > $OUT/i8mma.txt 2>&1
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_symm -s 1 -c 1 -o $OUT/oz_symm_cfg5 python tools/one_apply.py cfg5 128 0 1 > $OUT/ncu_cfg5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg5.csv python tools/one_apply.py cfg5 128 0 2 > $OUT/ncu_l5.log 2>&1
