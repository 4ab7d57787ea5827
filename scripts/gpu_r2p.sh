#!/bin/bash
# Session p: the cluster-resident small-factor tridiagonalisation -- GPU suite, sanitizer on small
# shapes, bench lines for mlp / r32 (small path) and r50 (panel path, unchanged).
OUT=gpurun_out/r2p; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 compute-sanitizer --tool memcheck python scripts/sanitize_small.py > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for c in mlp r32; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 300 compute-sanitizer --tool racecheck python scripts/sanitize_small.py > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
