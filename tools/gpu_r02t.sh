OUT=gpurun_out/r02t; mkdir -p $OUT
python -c "from paper_2101_12164_b200 import build as B; B.build()" > $OUT/build.log 2>&1
for ak in 2 3; do timeout 300 python tools/one_apply.py cfg2 128 $ak 20 >> $OUT/time.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/one_apply.py cfg2 128 3 3 > $OUT/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_oz_symm -c 1 -o $OUT/oz_symm python tools/one_apply.py cfg2 128 3 1 > $OUT/ncu2.log 2>&1
