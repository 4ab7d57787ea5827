#!/bin/bash
# Ozaki row-max change: eigen/ozaki/fullsize/poison tests, r50 line, per-launch times of the ozk_* kernels.
OUT=gpurun_out/${TAG:-ozk}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_eigen_trd.py tests/test_gpu_fullsize.py tests/test_gpu_ws_poison.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --config r50 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $OUT/bench_r50.json 2> $OUT/bench_r50.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ozk_ --csv --log-file $OUT/launches_ozk.csv \
  python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu.log 2>&1
python scripts/ncu_summary.py launches $OUT/launches_ozk.csv $OUT/launches_ozk.md
