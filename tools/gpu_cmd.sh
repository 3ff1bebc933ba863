OUT=gpurun_out
timeout 600 bash tools/ab.sh base hc3 base hc3 > $OUT/ab16.log 2>&1
