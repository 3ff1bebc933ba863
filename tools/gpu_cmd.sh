OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_dsl.py tests/test_gpu_dsl_multirank.py -x -q > $OUT/gt47.log 2>&1; echo "rc=$?" >> $OUT/gt47.log
python bench.py --steps 10 --no-cpu-baseline --no-validation --no-policy --no-boa --no-e2e > $OUT/b47.log 2>&1
