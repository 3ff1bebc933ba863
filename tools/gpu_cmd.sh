OUT=gpurun_out
L=$PWD/paper_1704_03329_b200
LJMD_LIB_A=$L/libljmd_rr0.so LJMD_LIB_B=$L/libljmd_rr2.so timeout 300 python tools/same_traj.py > $OUT/same35.log 2>&1
timeout 600 bash tools/ab.sh rr0 rr2 rr0 rr2 > $OUT/ab35.log 2>&1
compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_drive.py 2>&1 | tail -c 6000 > $OUT/r2_memcheck.log
compute-sanitizer --tool racecheck python tools/sanitize_drive.py 2>&1 | tail -c 6000 > $OUT/r2_racecheck.log
