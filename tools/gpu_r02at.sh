#!/bin/bash
# round-2 record on HEAD (after the k_oz_symm leading-slice skip): smoke, full GPU suite, bench (cfg5 +
# cfg2), reference arm, ncu full of k_oz_symm at cfg5, launch list of the cfg5 bench apply
set -u
OUT=gpurun_out/${1:-r02at}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_symm -s 1 -c 1 -o $OUT/oz_symm_cfg5 python tools/one_apply.py cfg5 128 0 1 > $OUT/ncu_cfg5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg5.csv python tools/one_apply.py cfg5 128 0 2 > $OUT/ncu_l5.log 2>&1
