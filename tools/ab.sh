# A/B of libljmd variants on C2: python bench.py per variant (force us per launch, PTS/s)
# usage: bash tools/ab.sh v0 v1 v2 ...
for v in "$@"; do
  LJMD_LIB=$PWD/paper_1704_03329_b200/libljmd_$v.so python bench.py --steps 30 --no-e2e --no-cpu-baseline --no-boa --no-dsl --no-policy --no-clocks 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['value']/1e9,4), 'force_us', round(d['roofline']['avg_launch_ms']*1e3,1), 'frac', round(d['roofline']['frac'],4), 'ms/step', round(d['ms_per_step'],3))"
done
