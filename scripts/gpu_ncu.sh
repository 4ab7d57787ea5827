#!/bin/bash
# ncu --set full captures of named kernels inside one bench run each.
# Usage: TAG=p1 SPECS="syrk_tc:0:2 trd_panel:5:1" CFG=r50 bash scripts/gpu_ncu.sh
TAG=${TAG:-prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for spec in $SPECS; do
  K=${spec%%:*}; rest=${spec#*:}; S=${rest%%:*}; C=${rest#*:}
  timeout ${NCU_TIMEOUT:-900} ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C \
    -o $OUT/prof_${K}_s$S python bench.py --config ${CFG:-r50} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > $OUT/ncu_${K}_s$S.log 2>&1
  echo "$K rc=$?" >> $OUT/ncu_rc.txt
done
