#!/bin/bash
# Ozaki GEMM bring-up: unit tests, micro-benchmark, eigen tests, full-size eigen parity, r50 bench.
OUT=gpurun_out/r2c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_ozaki.py -q -x -rf > $OUT/pytest_ozaki.log 2>&1; echo "rc=$?" >> $OUT/pytest_ozaki.log
timeout 300 python scripts/micro_ozaki.py > $OUT/micro_ozaki.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_eigen_trd.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -rf -s > $OUT/pytest_eigen.log 2>&1; echo "rc=$?" >> $OUT/pytest_eigen.log
timeout 600 python bench.py --config r50 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_r50.json 2> $OUT/bench_r50.err
