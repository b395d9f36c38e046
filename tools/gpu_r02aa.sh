#!/bin/bash
# round-2 record: full GPU suite, bench (cfg5 + cfg2), reference arm, ncu of k_oz_symm (cfg5), launch lists
set -u
OUT=gpurun_out/${1:-r02aa}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_symm -s 1 -c 1 -o $OUT/oz_symm_cfg5 python tools/one_apply.py cfg5 128 0 1 > $OUT/ncu_cfg5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_cfg2.csv python bench.py --config cfg2 --no-secondary --no-cpu-baseline --no-nystrom --no-analog --steps 2 --warmup 1 > $OUT/ncu_b2.log 2>&1
