#!/bin/bash
set -u
TAG=${1:-r02f}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bcg.py tests/test_gpu_bench_path.py tests/test_gpu_nystrom.py tests/test_gpu_edge.py tests/test_gpu_pcg.py -q -m gpu -rA -s -p no:cacheprovider > "$OUT/pytest.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest.log"
for cfg in cfg2 cfg2s; do
  for v in "NSP_APPLY_FIRST=0" "NSP_APPLY_FIRST=1"; do
    env $v timeout 300 python tools/ab_bcg.py $cfg 15 --analog >> "$OUT/ab.jsonl" 2>> "$OUT/ab.err"
  done
done
for v in "NSP_GRAM_CL=1" "NSP_GRAM_CL=8"; do
  env $v timeout 300 python tools/ab_bcg.py cfg2 15 >> "$OUT/ab_cl.jsonl" 2>> "$OUT/ab.err"
done
env NSP_GRAM_CL=1 timeout 600 python tools/ab_bcg.py cfg5 3 >> "$OUT/ab_cl.jsonl" 2>> "$OUT/ab.err"
env NSP_GRAM_CL=8 timeout 600 python tools/ab_bcg.py cfg5 3 >> "$OUT/ab_cl.jsonl" 2>> "$OUT/ab.err"
NSP_PRECS=2 NSP_PCG_WARM=0 NSP_GRAPH=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv \
      --log-file "$OUT/launches_pcg_cfg5.csv" python tools/time_pcg.py cfg5 1 > "$OUT/ncu_pcg_cfg5.log" 2>&1
