OUT=gpurun_out
timeout 300 python tools/same_env.py LJMD_FUSE 0 1 C1 > $OUT/same46.log 2>&1
for v in 0 1 0 1; do LJMD_FUSE=$v python bench.py --config C1 --steps 50 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl --no-e2e 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fuse=$v', d['value'], d['ms_per_step'])" >> $OUT/c1_46.log; done
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gt46.log 2>&1; echo "rc=$?" >> $OUT/gt46.log
