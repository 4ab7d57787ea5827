#!/bin/bash
# Diagnostic: per-phase trd_panel latency (timing build), then the normal build, eigen tests, bench.
OUT=gpurun_out/${TAG:-tim}; mkdir -p $OUT
KFAC_NVCC_EXTRA="-DKFAC_TRD_TIMING=1 $KFAC_NVCC_EXTRA" python -c "import __graft_entry__ as g; g.build()" > $OUT/build_tim.log 2>&1
timeout 300 python scripts/trd_timing.py 4609 > $OUT/t4609.txt 2>&1
rm -f paper_2007_00784_b200/libkfac.so
TAG=${TAG:-tim} TESTS="${TESTS:-tests/test_gpu_eigen_trd.py tests/test_gpu_parity.py}" bash scripts/gpu_quick.sh
