#!/bin/bash
# One GPU pass: gpu tests, smoke, the headline bench lines, the launch list and the full ncu capture.
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gputests.log 2>&1; echo "gputests rc=$?" >> $OUT/gputests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 bash tools/bench_all.sh > $OUT/bench_all.log 2>&1
timeout 1200 bash tools/profile_r2.sh > $OUT/profile.log 2>&1
ls -la $OUT
