#!/bin/bash
# Session f: two-stage reduction routed by default for dominant mid-size factors.
OUT=gpurun_out/r2f; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --config r50 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_r50.json 2> $OUT/bench_r50.err
timeout 600 python scripts/eig_scaling.py --config r50 > $OUT/eig_scaling_r50.jsonl 2>&1
timeout 600 python bench.py --config mlp --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_mlp.json 2> $OUT/bench_mlp.err
