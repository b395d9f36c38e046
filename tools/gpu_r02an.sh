#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02an}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
NSP_LIB=tools/variants/ozprof/libnsp.so timeout 600 python tools/one_apply.py cfg5 128 0 3 > $OUT/prof5.txt 2>&1
NSP_LIB=tools/variants/ozprof/libnsp.so timeout 300 python tools/one_apply.py cfg2 128 0 3 > $OUT/prof2.txt 2>&1
