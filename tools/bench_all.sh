#!/bin/bash
# bench lines behind profiles/r2_bench_*.json (run on the GPU box from the repo root)
OUT=gpurun_out
mkdir -p $OUT
last() { grep '^{' "$1" | tail -1 > "$2"; }
python bench.py > $OUT/b_c2.log 2>&1; last $OUT/b_c2.log $OUT/r2_bench_c2.json
python bench.py --check 1 --no-cpu-baseline --no-boa --no-dsl > $OUT/b_c2s.log 2>&1; last $OUT/b_c2s.log $OUT/r2_bench_c2_safe.json
for c in C1 C3 C4 C5; do
  python bench.py --config $c --steps 20 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl \
      > $OUT/b_$c.log 2>&1; last $OUT/b_$c.log $OUT/r2_bench_$(echo $c | tr C c).json
done
python bench.py --split-self --steps 20 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl --no-e2e \
    > $OUT/b_split.log 2>&1; last $OUT/b_split.log $OUT/r2_bench_c2_split_self.json
python bench.py --newton3 --steps 10 --no-cpu-baseline --no-validation --no-policy --no-boa --no-dsl --no-e2e \
    > $OUT/b_n3.log 2>&1; last $OUT/b_n3.log $OUT/r2_bench_c2_newton3.json
python bench.py --impl reference --steps 5 --warmup 1 > $OUT/b_ref.log 2>&1; last $OUT/b_ref.log $OUT/r2_bench_reference_c2.json
ls -la $OUT/r2_bench_*.json
