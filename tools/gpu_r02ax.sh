#!/bin/bash
# after the zero-slice skip: which part binds k_oz_symm - no-load diagnostics (bit 1: no A loads, 2: no B loads)
set -u
OUT=gpurun_out/${1:-r02ax}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
for d in 0 1 2 3 0; do echo "dbg $d" >> $OUT/time.txt; NSP_OZ_DBG=$d timeout 600 python tools/one_apply.py cfg5 128 0 10 >> $OUT/time.txt 2>&1; done
