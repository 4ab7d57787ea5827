#!/bin/bash
# Session gg close: poison tests, full GPU suite, smoke, bench lines (r50 default with e2e +
# cpu_baseline, mlp, r32, r101, inverse), r50 launch list, ncu of the factor SYRK and trd_panel,
# eigen projection.  Outputs under gpurun_out/$TAG.
OUT=gpurun_out/${TAG:-r2gg2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ws_poison.py tests/test_gpu_sbr.py -q -rA > $OUT/pytest_poison.log 2>&1; echo "rc=$?" >> $OUT/pytest_poison.log
timeout 1500 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_r50_default.json 2> $OUT/bench_r50_default.err
for c in mlp r32 r101; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --config r50 --variant inverse --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r50_inverse.json 2> $OUT/bench_r50_inverse.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_r50.csv \
  python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_list.log 2>&1
python scripts/ncu_summary.py launches $OUT/launches_r50.csv $OUT/launches_r50.md
for spec in "trd_panel:5:1" "syrk_tc_planes8:0:1"; do
  K=${spec%%:*}; rest=${spec#*:}; S=${rest%%:*}; C=${rest#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C \
    -o $OUT/prof_${K}_s$S python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > $OUT/ncu_${K}_s$S.log 2>&1
  python scripts/ncu_summary.py full $OUT/prof_${K}_s$S.ncu-rep $OUT/prof_${K}_s$S.md
done
timeout 600 python scripts/eig_scaling.py --config r50 > $OUT/eig_scaling_r50.jsonl 2>&1
