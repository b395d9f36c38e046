#!/bin/bash
# Round-2 second GPU call: new-kernel tests, A/B timings of the fused kernels, chol microbenchmark,
# ncu launch lists (cfg2, cfg5) and ncu --set full captures (SpMM, Gram, panel, fused pass, k_symm cfg5).
set -u
TAG=${1:-r02b}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "from paper_2101_12164_b200 import build as B; B.build()" > "$OUT/build.log" 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bcg.py tests/test_gpu_apply.py -q -m gpu -rA -s -p no:cacheprovider > "$OUT/pytest_kern.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_kern.log"
timeout 600 python -m pytest tests/test_gpu_bench_path.py -q -m gpu -rA -s -p no:cacheprovider > "$OUT/pytest_path.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_path.log"
timeout 120 ./tools/bench_chol16 > "$OUT/bench_chol16.txt" 2>&1
timeout 120 ./tools/bench_chol16_warp > "$OUT/bench_chol16_warp.txt" 2>&1
for cfg in cfg2; do
  for v in "NSP_FUSED_SXS=0 NSP_FUSED_PG=0 NSP_SPMM_V=1" "NSP_FUSED_SXS=1 NSP_FUSED_PG=0 NSP_SPMM_V=1" \
           "NSP_FUSED_SXS=1 NSP_FUSED_PG=1 NSP_SPMM_V=1" "NSP_FUSED_SXS=1 NSP_FUSED_PG=1 NSP_SPMM_V=2"; do
    env $v timeout 300 python tools/ab_bcg.py $cfg 15 --analog >> "$OUT/ab_$cfg.jsonl" 2>> "$OUT/ab.err"
  done
done
SHORT2="python bench.py --config cfg2 --steps 1 --warmup 3 --apply-reps 2 --no-cpu-baseline --no-secondary --no-nystrom"
$SHORT2 > "$OUT/short2_plain.log" 2>&1 && NSP_GRAPH=1 timeout 900 \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
      --log-file "$OUT/launches_cfg2.csv" $SHORT2 > "$OUT/ncu_launches_cfg2.log" 2>&1
for k in k_spmm2 k_panel_gram k_gram_partial k_gram_reduce k_chol16 k_panel_rows; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 30 -c 2 \
      -o "$OUT/full_cfg2_$k" $SHORT2 > "$OUT/ncu_full_cfg2_$k.log" 2>&1
done
SHORT5="python bench.py --config cfg5 --steps 1 --warmup 1 --apply-reps 2 --no-cpu-baseline --no-secondary --no-nystrom --no-analog"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_symm|k_spmm2" -s 8 -c 3 \
    -o "$OUT/full_cfg5" $SHORT5 > "$OUT/ncu_full_cfg5.log" 2>&1
NSP_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file "$OUT/launches_cfg5.csv" $SHORT5 > "$OUT/ncu_launches_cfg5.log" 2>&1
