#!/bin/bash
# Session w: launch lists of one r32 and one mlp step (which kernels carry the small configs).
OUT=gpurun_out/r2w; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for c in r32 mlp; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_$c.log 2>&1
  python scripts/ncu_summary.py launches $OUT/launches_$c.csv $OUT/launches_$c.md
done
