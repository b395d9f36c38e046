#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02aq}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py tests/test_gpu_pcg.py tests/test_gpu_nystrom.py -q -m gpu -x > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for v in 0 1; do echo "oz_symv $v" >> $OUT/time.txt; NSP_OZ_SYMV=$v NSP_PRECS=2 NSP_PCG_WARM=1 timeout 900 python tools/time_pcg.py cfg5 2 >> $OUT/time.txt 2>&1; NSP_OZ_SYMV=$v NSP_PRECS=2 timeout 300 python tools/time_pcg.py cfg2 5 >> $OUT/time.txt 2>&1; done
