#!/bin/bash
# One gpurun call: GPU parity tests, the default bench line, the ncu launch list of a short bench and
# one `ncu --set full` capture of the top kernel.  Usage (from the repo root, on the GPU box):
#   bash tools/gpu_round.sh [tag] [kernel-regex]
set -u
TAG=${1:-r01}
KREGEX=${2:-k_symm}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"; grep -m1 "model name" /proc/cpuinfo >> "$OUT/nproc.txt"; free -g >> "$OUT/nproc.txt"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke exit $?" >> "$OUT/smoke.log"
timeout 1500 python -m pytest tests -q -m gpu -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench exit $?" >> "$OUT/bench.err"
SHORT="python bench.py --steps 1 --warmup 3 --apply-reps 2 --no-cpu-baseline"
$SHORT > "$OUT/short_plain.log" 2>&1 && NSP_GRAPH=1 \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
      --log-file "$OUT/launches.csv" $SHORT > "$OUT/ncu_launches.log" 2>&1
echo "ncu launches exit $?" >> "$OUT/ncu_launches.log"
ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -s 40 -c 1 \
    -o "$OUT/prof_top" $SHORT > "$OUT/ncu_full.log" 2>&1
echo "ncu full exit $?" >> "$OUT/ncu_full.log"
