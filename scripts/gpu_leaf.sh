#!/bin/bash
# D&C leaf-size experiment: eigen tests + mlp / r32 / r50 lines for KFAC_LEAF = 16 (then default).
OUT=gpurun_out/${TAG:-leaf}; mkdir -p $OUT
export KFAC_NVCC_EXTRA="-DKFAC_LEAF=16"
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_16.log 2>&1
timeout 600 python -m pytest tests/test_gpu_eigen_trd.py tests/test_gpu_parity.py -q -x -k "compute_eigen or divide or mlp or r32" > $OUT/pytest_16.log 2>&1; echo "rc=$?" >> $OUT/pytest_16.log
for c in mlp r32 r50; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_${c}_16.json 2> $OUT/bench_${c}_16.err
done
unset KFAC_NVCC_EXTRA
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_default.log 2>&1
