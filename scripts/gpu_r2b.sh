#!/bin/bash
# Round 2 session b: whole GPU suite, bench with graph replay, launch list, KL-clip ncu captures.
OUT=gpurun_out/r2b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1; echo "rc=$?" >> $OUT/build_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --config r50 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_r50.json 2> $OUT/bench_r50.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_r50.csv \
  python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > $OUT/ncu_list.log 2>&1
TAG=r2b SPECS="kl_dot:1:1 kl_scale:1:1" bash scripts/gpu_ncu.sh
