# Refresh profiles/: bench line, reference arm, ncu launch list, ncu --set full of the force
# kernel inside bench.py and of the auxiliary kernels (profiles/drive.py).
set -x
python bench.py > gpurun_out/r1_bench_c2.json 2> gpurun_out/bench_stderr.log
python bench.py --newton3 --no-e2e --no-cpu-baseline --no-boa --no-dsl > gpurun_out/r1_bench_c2_newton3.json 2>/dev/null
python bench.py --impl reference --steps 10 --warmup 1 > gpurun_out/r1_bench_reference_c2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-boa --no-dsl --no-clocks > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'k_force' --launch-skip 40 --launch-count 8 -o gpurun_out/r1_force_kernels python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-boa --no-dsl --no-clocks > gpurun_out/ncu_force.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'k_build_nlist|k_list_rr|k_ghost_flat|k_cell_sort|k_wrap_bin|k_boa|k_cna|ljmd_dsl|k_force_half|k_vv' -c 14 -o gpurun_out/r1_aux_kernels python profiles/drive.py > gpurun_out/ncu_aux.log 2>&1
ls -la gpurun_out
