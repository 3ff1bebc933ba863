#!/bin/bash
# per-kernel durations (ncu launch list, cold cache, serialised) of C2 init + one 20-step cycle
# for each library variant: bash tools/klist.sh v1 v2 ...   -> gpurun_out/kl_<v>.csv + summary
for v in "$@"; do
  LJMD_LIB=$PWD/paper_1704_03329_b200/libljmd_$v.so ncu --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/kl_$v.csv python tools/build_drive.py 1 > /dev/null 2>&1
  python tools/klsum.py gpurun_out/kl_$v.csv $v
done
