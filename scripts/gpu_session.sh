#!/bin/bash
# Full GPU session: tests, smoke, bench lines, ncu launch list + one full capture.
# Usage: TAG=r1 bash scripts/gpu_session.sh   (outputs under gpurun_out/$TAG)
TAG=${TAG:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -rA --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
fi
for c in ${BENCH_CONFIGS:-r50}; do
  timeout 1500 python bench.py --config $c ${BENCH_ARGS:---steps 3 --warmup 2} > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
if [ -n "$PROFILE" ]; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-12000} --csv \
    --log-file $OUT/launches_r50.csv python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_list.log 2>&1
  for K in $PROFILE; do
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-1} -c 1 \
      -o $OUT/prof_$K python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_$K.log 2>&1
  done
fi
