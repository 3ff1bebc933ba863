OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gt44.log 2>&1; echo "rc=$?" >> $OUT/gt44.log
for c in C1 C1; do python bench.py --config $c --steps 50 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl --no-e2e 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['ms_per_step'])" >> $OUT/b44.log; done
timeout 600 bash tools/abenv.sh LJMD_NONE 0 0 >> $OUT/b44.log 2>&1
