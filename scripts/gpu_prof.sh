#!/bin/bash
# Profiling session: launch list (gpu__time_duration) + one full ncu capture of a named kernel.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CFG=${CFG:-r32}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-3000} --csv \
  --log-file gpurun_out/launches_${CFG}.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_list_${CFG}.log 2>&1
if [ -n "$KERNEL" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KERNEL -s ${SKIP:-2} -c ${COUNT:-1} \
    -o gpurun_out/prof_${CFG}_${KERNEL} python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${CFG}.log 2>&1
fi
