OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c2 or C2" > $OUT/gt38.log 2>&1; echo "rc=$?" >> $OUT/gt38.log
