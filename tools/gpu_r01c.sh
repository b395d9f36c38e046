#!/bin/bash
# SYMM apply round: parity tests (both apply kernels), block CG, bench with CW 32 / 64, ncu of k_symm
OUT=gpurun_out/r01c; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x -k "apply or bcg or nystrom" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
NSP_CW=32 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_cw32.json 2> $OUT/bench_cw32.err
NSP_CW=64 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_cw64.json 2> $OUT/bench_cw64.err
SHORT="python bench.py --steps 1 --warmup 3 --apply-reps 2 --no-cpu-baseline"
$SHORT > $OUT/short_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_symm -s 40 -c 1 -o $OUT/prof_symm $SHORT > $OUT/ncu_full.log 2>&1
echo "ncu exit $?" >> $OUT/ncu_full.log
