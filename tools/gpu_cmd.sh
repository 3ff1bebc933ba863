OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/gt31.log 2>&1; echo "rc=$?" >> $OUT/gt31.log
timeout 600 bash tools/abenv.sh LJMD_PERSIST 0 1 0 1 > $OUT/ab31.log 2>&1
