#!/bin/bash
# Session bb: ncu --set full of the small-d factor SYRK (r32) and of the small-factor reduction (mlp).
OUT=gpurun_out/${TAG:-r2bb}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:syrk_small -c 1 -o $OUT/prof_syrk_small_r32 \
  python bench.py --config r32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_syrk_small.log 2>&1
python scripts/ncu_summary.py full $OUT/prof_syrk_small_r32.ncu-rep $OUT/prof_syrk_small_r32.md
