for v in 0 1 2 3 0 3; do
  LJMD_LIB=$PWD/paper_1704_03329_b200/libljmd_v$v.so python bench.py --steps 30 --no-e2e --no-cpu-baseline --no-boa --no-dsl --no-clocks 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('v$v', round(d['value']/1e9,4), round(d['roofline']['avg_launch_ms']*1e3,1), round(d['roofline']['frac'],4))"
done
LJMD_LIB=$PWD/paper_1704_03329_b200/libljmd_v3.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
