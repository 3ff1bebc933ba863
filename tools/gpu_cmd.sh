OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gt10.log 2>&1; echo "rc=$?" >> $OUT/gt10.log
python bench.py --config C1 --steps 50 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl > $OUT/b10_c1.log 2>&1
python bench.py --steps 30 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl > $OUT/b10_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/c1_b10.csv python tools/c1_drive.py > /dev/null 2>&1
python tools/klsum.py $OUT/c1_b10.csv c1 > $OUT/c1_b10.txt
