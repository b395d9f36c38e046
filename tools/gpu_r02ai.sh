#!/bin/bash
# record: full GPU suite, bench, ncu of k_oz_symm (cfg5), smoke()
set -u
OUT=gpurun_out/${1:-r02ai}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "exit $?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_symm -s 1 -c 1 -o $OUT/oz_symm_cfg5 python tools/one_apply.py cfg5 128 0 1 > $OUT/ncu_cfg5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_cfg5.csv python bench.py --no-secondary --no-cpu-baseline --no-nystrom --no-analog --steps 1 --warmup 1 --apply-reps 1 > $OUT/ncu_b5.log 2>&1
