#!/bin/bash
# round-2 full-size record on the latest code (INT8 a2+a3): every BASELINE config's setup, memory, apply,
# block CG to tol; Nystrom + outer PCG (S~_1, M_2, M_A-DEF2) at full size
set -u
OUT=gpurun_out/${1:-r02au}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 1500 python tools/fullsize.py cfg2 cfg3 cfg4 cfg5 > $OUT/fullsize.jsonl 2> $OUT/fullsize.err
NSP_PRECS=1,2,3 timeout 1500 python tools/fullsize.py --pcg cfg2 cfg5 > $OUT/fullsize_pcg.jsonl 2> $OUT/fullsize_pcg.err
