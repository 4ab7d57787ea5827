#!/bin/bash
# Factor-SYRK A/B: CTA order (tile-major vs row-chunk-major) and row chunk size; r50 / r101 / r32
# lines per variant plus the factor parity tests.  VARIANTS: name:macros entries separated by ';'.
OUT=gpurun_out/${TAG:-syrk}; mkdir -p $OUT
IFS=';' read -ra VS <<< "${VARIANTS:-tile:-DKFAC_SYRK_SPLIT_MAJOR=0;split:;split8k:-DKFAC_SYRK_CHUNK=8192}"
for V in "${VS[@]}"; do
  name=${V%%:*}; export KFAC_NVCC_EXTRA="${V#*:}"
  python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$name.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "factor or full_size or r32" > $OUT/pytest_$name.log 2>&1; echo "rc=$?" >> $OUT/pytest_$name.log
  for c in ${CONFIGS:-r50 r32}; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $OUT/bench_${c}_$name.json 2> $OUT/bench_${c}_$name.err
  done
  if [ -n "$NCU" ]; then
    timeout 600 ncu --set full --clock-control none -k regex:syrk_tc_planes8 -s 0 -c 1 -o $OUT/prof_syrk_$name \
      python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_$name.log 2>&1
    python scripts/ncu_summary.py full $OUT/prof_syrk_$name.ncu-rep $OUT/prof_syrk_$name.md
  fi
done
unset KFAC_NVCC_EXTRA
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_default.log 2>&1
