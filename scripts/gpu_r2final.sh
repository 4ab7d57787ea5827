#!/bin/bash
# Round-2 end-of-session evidence: full GPU suite, smoke, bench lines (default r50 with e2e +
# cpu_baseline, mlp, r32, r101, r50 inverse / factored variants, reference arm), launch list,
# eigen scaling projection.  Outputs under gpurun_out/$TAG.
TAG=${TAG:-r2final}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_r50_default.json 2> $OUT/bench_r50_default.err
for c in mlp r32 r101; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
for v in inverse factored; do
  timeout 900 python bench.py --config r50 --variant $v --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r50_$v.json 2> $OUT/bench_r50_$v.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_r50.csv \
  python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_list.log 2>&1
python scripts/ncu_summary.py launches $OUT/launches_r50.csv $OUT/launches_r50.md
timeout 600 python scripts/eig_scaling.py --config r50 > $OUT/eig_scaling_r50.jsonl 2>&1
timeout 300 python scripts/sbr_time.py 785 1025 2305 4609 > $OUT/lone_factors.jsonl 2>&1
