#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02ap}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_nystrom.py tests/test_gpu_bcg.py tests/test_gpu_multirank.py tests/test_gpu_edge.py -q -m gpu -x > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for v in 0 1; do echo "cheb3 $v" >> $OUT/time.txt; NSP_CHEB3=$v NSP_PRECS=2 NSP_PCG_WARM=1 timeout 900 python tools/time_pcg.py cfg5 2 >> $OUT/time.txt 2>&1; done
for v in 0 1; do echo "cheb3 $v" >> $OUT/time_ag.txt; NSP_CHEB3=$v timeout 900 python bench.py --no-secondary --no-cpu-baseline --no-nystrom --steps 3 --warmup 3 > $OUT/bench_$v.json 2>> $OUT/time_ag.txt; done
