OUT=gpurun_out
timeout 900 bash tools/klist.sh bl0 bl1 > $OUT/kl52.log 2>&1
timeout 600 bash tools/ab.sh bl0 bl1 bl0 bl1 > $OUT/ab52.log 2>&1
