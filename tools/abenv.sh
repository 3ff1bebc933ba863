# A/B of an environment switch on C2: bash tools/abenv.sh VAR v1 v2 ...
var=$1; shift
for v in "$@"; do
  env $var=$v python bench.py --steps 30 --no-e2e --no-cpu-baseline --no-boa --no-dsl --no-policy --no-clocks --no-validation 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$var=$v', round(d['value']/1e9,4), 'force_us', round(d['roofline']['avg_launch_ms']*1e3,1), 'frac', round(d['roofline']['frac'],4), 'ms/step', round(d['ms_per_step'],3))"
done
