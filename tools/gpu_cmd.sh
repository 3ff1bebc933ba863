OUT=gpurun_out
timeout 300 python tools/same_env.py LJMD_SMALL_BUILD 0 1 C1 > $OUT/same40.log 2>&1
for v in 0 1 0 1; do LJMD_SMALL_BUILD=$v python bench.py --config C1 --steps 50 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl --no-e2e 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('small=$v', d['value'], d['ms_per_step'])" >> $OUT/c1_40.log; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/c1_40.csv python tools/c1_drive.py > /dev/null 2>&1
python tools/klsum.py $OUT/c1_40.csv c1 > $OUT/c1_40.txt
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/gt40.log 2>&1; echo "rc=$?" >> $OUT/gt40.log
