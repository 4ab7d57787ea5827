#!/bin/bash
OUT=gpurun_out/r2e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python scripts/micro_ozaki.py > $OUT/micro_ozaki.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --config r50 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_r50.json 2> $OUT/bench_r50.err
