#!/bin/bash
set -u
TAG=${1:-r02h}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
timeout 900 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_nystrom.py -q -m gpu -rA -p no:cacheprovider > "$OUT/pytest.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest.log"
for v in "NSP_CHEB_G=2 NSP_SPMV_G=8" "NSP_CHEB_G=4 NSP_SPMV_G=8" "NSP_CHEB_G=4 NSP_SPMV_G=4" "NSP_CHEB_G=4 NSP_SPMV_G=2"; do
  echo "$v" >> "$OUT/time_pcg_cfg5.txt"
  env $v NSP_PRECS=2 NSP_PCG_WARM=1 timeout 600 python tools/time_pcg.py cfg5 2 >> "$OUT/time_pcg_cfg5.txt" 2>&1
  echo "$v" >> "$OUT/time_pcg_cfg2.txt"
  env $v NSP_PRECS=2,1 timeout 600 python tools/time_pcg.py cfg2 5 >> "$OUT/time_pcg_cfg2.txt" 2>&1
done
NSP_PRECS=2 NSP_PCG_WARM=0 NSP_GRAPH=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv \
      --log-file "$OUT/launches_pcg_cfg5.csv" python tools/time_pcg.py cfg5 1 > "$OUT/ncu_pcg_cfg5.log" 2>&1
