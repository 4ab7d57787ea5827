#!/bin/bash
# Session s: ncu --set full of the small-factor reduction (d = 145 on one CTA, d = 785 on a 13-CTA
# cluster) with source correlation; the lone-factor times of the symv-rows templated panel kernel.
OUT=gpurun_out/r2s; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for n in 145 785; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:trd_small -c 1 -o $OUT/small_$n \
    python scripts/sbr_time.py $n > $OUT/ncu_$n.log 2>&1
done
timeout 300 python scripts/sbr_time.py 1153 2305 4609 > $OUT/lone_big.jsonl 2>&1
timeout 600 python bench.py --config r50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r50.json 2> $OUT/bench_r50.err
timeout 600 python scripts/eig_scaling.py --config r50 > $OUT/eig_scaling_r50.jsonl 2>&1
