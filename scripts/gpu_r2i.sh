#!/bin/bash
# ncu --set full captures (one launch each) of the dominant kernels of an r50 step at HEAD.
OUT=gpurun_out/r2i; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for spec in "ozk_slice:20:1" "ozk_rowmax:20:1" "ozk_gemm:20:1" "trd_panel:5:1" "syrk_tc_planes8:0:1" "gemm_tc_planes:2:1" "gemm64_direct:40:1" "dc_secular:0:1"; do
  K=${spec%%:*}; rest=${spec#*:}; S=${rest%%:*}; C=${rest#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C \
    -o $OUT/prof_${K}_s$S python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > $OUT/ncu_${K}_s$S.log 2>&1
  echo "$K rc=$?" >> $OUT/ncu_rc.txt
done
