#!/bin/bash
# full GPU suite + bench (cfg5 headline + cfg2 secondary) + ncu capture of k_oz_symm at cfg5
set -u
OUT=gpurun_out/${1:-r02v}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_oz_symm -s 2 -c 1 -o $OUT/oz_symm_cfg5 python tools/one_apply.py cfg5 128 0 1 > $OUT/ncu_cfg5.log 2>&1
