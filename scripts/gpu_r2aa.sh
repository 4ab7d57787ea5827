#!/bin/bash
# Session aa: small-d factor SYRK entry loop + small-factor reduction block sums: parity tests, GPU
# suite, r32 / mlp lines, r32 launch list.
OUT=gpurun_out/${TAG:-r2aa}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "factors or r32 or mlp or compute_eigen" > $OUT/pytest_quick.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for c in r32 mlp; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_r32.csv \
  python bench.py --config r32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_r32.log 2>&1
python scripts/ncu_summary.py launches $OUT/launches_r32.csv $OUT/launches_r32.md
