#!/bin/bash
# the executed-products roofline (nsp_ozaki_stats): INT8 tests incl. the work-count test, smoke, bench
set -u
OUT=gpurun_out/${1:-r02av}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_apply.py tests/test_setup_validation.py -q -m gpu -x -s > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
