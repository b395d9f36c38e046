#!/bin/bash
# bench with the double-buffered e2e loop
set -u
OUT=gpurun_out/${1:-r02ay}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
