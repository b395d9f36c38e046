#!/bin/bash
# Round-2 third GPU call: full GPU suite (incl. the sharded Nystrom / PCG tests), default bench line,
# cfg5 A/B of the fused tall-skinny kernels.
set -u
TAG=${1:-r02c}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke exit $?" >> "$OUT/smoke.log"
timeout 2400 python -m pytest tests -q -m gpu -rA -s -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench exit $?" >> "$OUT/bench.err"
for v in "NSP_FUSED_SXS=0 NSP_FUSED_PG=0" "NSP_FUSED_SXS=1 NSP_FUSED_PG=1"; do
  env $v timeout 600 python tools/ab_bcg.py cfg5 3 >> "$OUT/ab_cfg5.jsonl" 2>> "$OUT/ab.err"
done
for v in "NSP_SPMM_V=1" "NSP_SPMM_V=2"; do
  env $v timeout 300 python tools/ab_bcg.py cfg2 15 >> "$OUT/ab_cfg2.jsonl" 2>> "$OUT/ab.err"
done
SHORT2="python bench.py --config cfg2 --steps 1 --warmup 3 --apply-reps 2 --no-cpu-baseline --no-secondary --no-nystrom"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_spmm2" -s 30 -c 2 \
    -o "$OUT/full_cfg2_k_spmm2" $SHORT2 > "$OUT/ncu_full_cfg2_k_spmm2.log" 2>&1
