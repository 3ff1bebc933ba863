OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gt43.log 2>&1; echo "rc=$?" >> $OUT/gt43.log
python bench.py --config C1 --steps 50 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl > $OUT/b43_c1.log 2>&1
python bench.py --steps 30 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl > $OUT/b43_c2.log 2>&1
