#!/bin/bash
set -u
TAG=${1:-r02g}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke exit $?" >> "$OUT/smoke.log"
timeout 2400 python -m pytest tests -q -m gpu -rA -s -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
for v in "NSP_CHEB_FUSED=0" "NSP_CHEB_G=4" "NSP_CHEB_G=8" "NSP_CHEB_G=16"; do
  echo "$v" >> "$OUT/time_pcg_cfg5.txt"
  env $v NSP_PRECS=2 NSP_PCG_WARM=1 timeout 600 python tools/time_pcg.py cfg5 2 >> "$OUT/time_pcg_cfg5.txt" 2>&1
done
timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench exit $?" >> "$OUT/bench.err"
