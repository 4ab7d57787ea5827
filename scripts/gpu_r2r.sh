#!/bin/bash
# Session r: small-factor reduction with buffered outputs: eigen tests, lone times + launch list,
# GPU suite, mlp / r32 lines.
OUT=gpurun_out/${TAG:-r2r}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_eigen_trd.py tests/test_gpu_parity.py -q -x -k "compute_eigen or mlp" > $OUT/pytest_quick.log 2>&1; echo "rc=$?" >> $OUT/pytest_quick.log
timeout 300 python scripts/sbr_time.py 145 289 577 785 > $OUT/lone_small.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_small.csv python scripts/sbr_time.py 145 577 785 > $OUT/ncu_small.log 2>&1
python scripts/ncu_summary.py launches $OUT/launches_small.csv $OUT/launches_small.md
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for c in mlp r32; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
