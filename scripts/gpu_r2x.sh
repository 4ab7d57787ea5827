#!/bin/bash
# Session x: small-d factor SYRK -- factor parity tests, GPU suite, r32 / mlp lines and launch lists.
OUT=gpurun_out/r2x; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/pytest_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity.log
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for c in r32 mlp; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_$c.log 2>&1
  python scripts/ncu_summary.py launches $OUT/launches_$c.csv $OUT/launches_$c.md
done
