#!/bin/bash
# Round 2 first GPU session: full-size parity tests + baseline bench.
OUT=gpurun_out/r2a; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_dist.py -m gpu -q -s -rA > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
timeout 600 python bench.py --config r50 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_r50.json 2> $OUT/bench_r50.err
