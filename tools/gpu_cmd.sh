OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gt13.log 2>&1; echo "rc=$?" >> $OUT/gt13.log
for bf in 1 0 1 0; do
LJMD_BFIRST=$bf python bench.py --split-self --steps 20 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl --no-e2e 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bfirst=$bf', d['value'], d['ms_per_step'])" >> $OUT/bf13.log
done
LJMD_GRAPHS=0 LJMD_SPLIT_SELF=1 timeout 300 python tools/kprof.py 5 > $OUT/kp13_split.log 2>&1
