#!/bin/bash
# Build-flag experiment: for each entry of $VARIANTS (a KFAC_NVCC_EXTRA string, "default" for none)
# build libkfac, run the eigen parity tests, one r50 bench line and lone-factor times.
# Usage: TAG=x VARIANTS="default;-DKFAC_SYMV_ROWS=24" bash scripts/gpu_variants.sh
OUT=gpurun_out/${TAG:-var}; mkdir -p $OUT
IFS=';' read -ra VS <<< "${VARIANTS:-default}"
j=0
for V in "${VS[@]}"; do
  if [ "$V" = "default" ]; then unset KFAC_NVCC_EXTRA; else export KFAC_NVCC_EXTRA="$V"; fi
  echo "$j: $V" >> $OUT/variants.txt
  python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$j.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_eigen_trd.py tests/test_gpu_fullsize.py -q -x > $OUT/pytest_$j.log 2>&1; echo "rc=$?" >> $OUT/pytest_$j.log
  timeout 600 python bench.py --config r50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r50_$j.json 2> $OUT/bench_r50_$j.err
  timeout 300 python scripts/sbr_time.py ${LONE:-1153 2305 4609} > $OUT/lone_$j.jsonl 2>&1
  j=$((j+1))
done
unset KFAC_NVCC_EXTRA
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_default.log 2>&1
