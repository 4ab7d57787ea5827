#!/bin/bash
# L2 residency of the lone d = 4609 tridiagonalisation: one ncu --set full capture of a mid panel.
OUT=gpurun_out/${TAG:-l2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:trd_panel -s ${SKIP:-30} -c 1 -o $OUT/lone4609 -f \
  python scripts/trd_timing.py 4609 > $OUT/ncu.log 2>&1
echo "ncu rc=$?" >> $OUT/ncu.log
