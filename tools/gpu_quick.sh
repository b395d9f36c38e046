#!/bin/bash
# quick GPU check: parity tests (-k filter) + one bench line.  Usage: bash tools/gpu_quick.sh TAG "kexpr"
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x -k "$2" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
