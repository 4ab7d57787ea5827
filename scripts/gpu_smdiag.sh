#!/bin/bash
# Small-factor reduction diagnostic: lone small-factor times with the matrix passes skipped
# (-DKFAC_SM_NOWORK=1, wrong results: timing of the per-column fixed cost only) and as built.
OUT=gpurun_out/${TAG:-smdiag}; mkdir -p $OUT
for V in "-DKFAC_SM_NOWORK=1" "default"; do
  if [ "$V" = "default" ]; then unset KFAC_NVCC_EXTRA; else export KFAC_NVCC_EXTRA="$V"; fi
  python -c "import __graft_entry__ as g; g.build()" > $OUT/build_${V//[^a-zA-Z0-9]/_}.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${V//[^a-zA-Z0-9]/_}.csv \
    python scripts/sbr_time.py 145 577 785 > /dev/null 2>&1
done
unset KFAC_NVCC_EXTRA
