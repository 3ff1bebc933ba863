OUT=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/gt5.log 2>&1; echo "rc=$?" >> $OUT/gt5.log
timeout 600 bash tools/ab.sh hicut nohicut hicut nohicut > $OUT/ab5.log 2>&1
timeout 600 bash tools/klist.sh hicut nohicut > $OUT/kl5.log 2>&1
