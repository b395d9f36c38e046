#!/bin/bash
# round 2, final record on HEAD: ncu launch list of the cfg5 bench step; ncu --set full of the Gram and panel
# kernels at cfg5 (DMMA utilisation of the tall-skinny contractions at the headline size)
OUT=gpurun_out/bc
mkdir -p $OUT
B="python bench.py --no-secondary --no-cpu-baseline --no-nystrom --no-analog --steps 1 --warmup 1 --apply-reps 1"
$B > $OUT/bench_plain.json 2> $OUT/bench_plain.err; echo plain $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_cfg5.csv $B > $OUT/ncu_b5.log 2>&1; echo list $?
python tools/ncu_summary.py $OUT/launches_bench_cfg5.csv > $OUT/launches_bench_cfg5_summary.txt; head -12 $OUT/launches_bench_cfg5_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_partial -s 3 -c 2 -o $OUT/gram_cfg5 $B > $OUT/ncu_gram.log 2>&1; echo gram $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_panel_rows -s 3 -c 1 -o $OUT/panel_cfg5 $B > $OUT/ncu_panel.log 2>&1; echo panel $?
ls -la $OUT
