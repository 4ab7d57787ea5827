#!/bin/bash
# Session t: lone-factor and scaling-projection times with the lone-launch symv geometry, r50 line,
# eigen GPU tests.
OUT=gpurun_out/${TAG:-r2t}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_eigen_trd.py tests/test_gpu_fullsize.py tests/test_gpu_sbr.py -q -x > $OUT/pytest_eigen.log 2>&1; echo "rc=$?" >> $OUT/pytest_eigen.log
timeout 300 python scripts/sbr_time.py 1153 2305 4609 > $OUT/lone_big.jsonl 2>&1
timeout 600 python scripts/eig_scaling.py --config r50 > $OUT/eig_scaling_r50.jsonl 2>&1
timeout 600 python bench.py --config r50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r50.json 2> $OUT/bench_r50.err
