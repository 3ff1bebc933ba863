#!/bin/bash
# The captures behind profiles/r2_* (run on the GPU box from the repo root):
#   bash tools/profile_r2.sh            -> gpurun_out/r2_*.{csv,ncu-rep,log}
# then, here: python profiles/extract_r2.py gpurun_out/r2_full.ncu-rep profiles/r2_kernels.json \
#                 --traffic profiles/force_traffic.json
set -x
OUT=gpurun_out
mkdir -p $OUT
# 1. launch list of the bench command (cold-cache, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/r2_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-boa --no-dsl --no-policy --no-validation \
    --no-clocks > $OUT/r2_launches_bench.log 2>&1
# 2. full sets: C2 init + one 20-step cycle (3 force launches incl. the two energy variants, the
#    list build and bank-aware pass, the binning and integration kernels)
ncu --set full --import-source on --clock-control none \
    -k regex:"k_force|k_build_nlist|k_list_rr|k_wrap_bin|k_cell_sort|k_kick_drift|k_maxdisp|k_ghost_refresh|k_scatter|k_tile_rows|k_img_build|k_finalize" \
    -s 12 -c 24 -o $OUT/r2_full python tools/build_drive.py 1 > $OUT/r2_full.log 2>&1
python profiles/extract_r2.py $OUT/r2_full.ncu-rep $OUT/r2_force_kernels_summary.json --traffic $OUT/force_traffic.json \
    > $OUT/r2_full_extract.log 2>&1 && rm -f $OUT/r2_full.ncu-rep   # gpurun copies back <= 64 MiB
# 3. the binning / list / integration kernels of one rebuild cycle
ncu --set full --import-source on --clock-control none \
    -k regex:"k_build_nlist|k_list_rr|k_wrap_bin|k_cell_sort|k_kick_drift|k_maxdisp|k_ghost_refresh|k_scatter|k_tile_rows|k_img_build" \
    -c 14 -o $OUT/r2_aux python tools/build_drive.py 1 > $OUT/r2_aux.log 2>&1
python profiles/extract_r2.py $OUT/r2_aux.ncu-rep $OUT/r2_aux_kernels_summary.json > $OUT/r2_aux_extract.log 2>&1 \
    && rm -f $OUT/r2_aux.ncu-rep
# 4. sanitizers: profiles/r2_memcheck.log and r2_racecheck.log were taken earlier in round 2;
#    compute-sanitizer has since been closed on the GPU pool (runs under it left GPUs needing a
#    reset), so it is no longer run here
