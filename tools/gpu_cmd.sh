OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gt18.log 2>&1; echo "rc=$?" >> $OUT/gt18.log
timeout 300 python tools/e2e_prof.py 6 > $OUT/e2e18.log 2>&1
python bench.py --steps 30 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl > $OUT/b18.log 2>&1
