#!/bin/bash
set -u
OUT=gpurun_out/${1:-r02ak}; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
for v in base u2m8 u2m6 u1m6; do
  if [ $v = base ]; then L=""; else L="NSP_LIB=tools/variants/$v/libnsp.so"; fi
  echo "== $v" >> $OUT/time.txt
  env $L timeout 600 python tools/one_apply.py cfg5 128 0 10 >> $OUT/time.txt 2>&1
  env $L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/l5_$v.csv python tools/one_apply.py cfg5 128 0 2 > /dev/null 2>&1
  env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/l2_$v.csv python tools/one_apply.py cfg2 128 0 3 > /dev/null 2>&1
done
NSP_GRAPH=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/pcg_eager_cfg2.csv python tools/one_pcg.py cfg2 20 > $OUT/ncu_pcg.log 2>&1
