OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gt50.log 2>&1; echo "rc=$?" >> $OUT/gt50.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke50.log 2>&1
timeout 1500 bash tools/bench_all.sh > $OUT/bench_all50.log 2>&1
