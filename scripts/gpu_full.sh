#!/bin/bash
# Round-end style GPU session: full gpu tests, smoke, default bench line (r50, e2e + cpu_baseline),
# other configs, reference arm.  Outputs under gpurun_out/$TAG.
TAG=${TAG:-full}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_r50_default.json 2> $OUT/bench_r50_default.err
for c in ${CONFIGS:-mlp r32 r101}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
