#!/bin/bash
# End-of-round refresh at HEAD after the last small-config changes: GPU suite, smoke, r50 default line
# (e2e + cpu_baseline + parity), mlp / r32 lines, r32 launch list, eigen projection.
OUT=gpurun_out/${TAG:-r2final2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_r50_default.json 2> $OUT/bench_r50_default.err
for c in mlp r32; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_r32.csv \
  python bench.py --config r32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_r32.log 2>&1
python scripts/ncu_summary.py launches $OUT/launches_r32.csv $OUT/launches_r32.md
timeout 600 python scripts/eig_scaling.py --config r50 > $OUT/eig_scaling_r50.jsonl 2>&1
