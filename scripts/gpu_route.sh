#!/bin/bash
# Two-stage routing experiment: r50 bench + eigen scaling projection per build-macro variant.
OUT=gpurun_out/${TAG:-route}; mkdir -p $OUT
# VARIANTS: name:macros entries separated by ';'
IFS=';' read -ra VS <<< "${VARIANTS:-base:;big:-DKFAC_SBR_SHARE=0.2 -DKFAC_SBR_MAXN=5000;dom:-DKFAC_SBR_MAXN=5000}"
for V in "${VS[@]}"; do
  name=${V%%:*}; export KFAC_NVCC_EXTRA="${V#*:}"
  python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$name.log 2>&1
  timeout 600 python bench.py --config r50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $OUT/bench_r50_$name.json 2> $OUT/bench_r50_$name.err
  timeout 300 python scripts/eig_scaling.py --config r50 > $OUT/eig_scaling_$name.jsonl 2>&1
  if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests/test_gpu_sbr.py tests/test_gpu_fullsize.py -q -x > $OUT/pytest_$name.log 2>&1; echo "rc=$?" >> $OUT/pytest_$name.log; fi
done
unset KFAC_NVCC_EXTRA
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_default.log 2>&1
