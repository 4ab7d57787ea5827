#!/bin/bash
# Round-2 end-of-session evidence: full GPU suite, smoke, bench lines (default r50 with e2e +
# cpu_baseline + parity, mlp, r32, r101, r152, r50 inverse / factored variants, reference arm),
# launch list, ncu --set full of the dominant kernels, eigen scaling projection, lone factors.
# Outputs under gpurun_out/$TAG.
TAG=${TAG:-r2final}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_r50_default.json 2> $OUT/bench_r50_default.err
for c in mlp r32 r101 r152; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
for v in inverse factored; do
  timeout 900 python bench.py --config r50 --variant $v --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r50_$v.json 2> $OUT/bench_r50_$v.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_r50.csv \
  python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_list.log 2>&1
python scripts/ncu_summary.py launches $OUT/launches_r50.csv $OUT/launches_r50.md
for spec in "trd_panel:5:1" "ozk_gemm:20:1" "syrk_tc_planes8:0:1" "gemm_tc_planes:2:1"; do
  K=${spec%%:*}; rest=${spec#*:}; S=${rest%%:*}; C=${rest#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C \
    -o $OUT/prof_${K}_s$S python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > $OUT/ncu_${K}_s$S.log 2>&1
  python scripts/ncu_summary.py full $OUT/prof_${K}_s$S.ncu-rep $OUT/prof_${K}_s$S.md
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trd_small -c 1 -o $OUT/prof_trd_small_mlp \
  python bench.py --config mlp --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_trd_small.log 2>&1
python scripts/ncu_summary.py full $OUT/prof_trd_small_mlp.ncu-rep $OUT/prof_trd_small_mlp.md
timeout 600 python scripts/eig_scaling.py --config r50 > $OUT/eig_scaling_r50.jsonl 2>&1
timeout 300 python scripts/sbr_time.py 785 1153 2305 4609 > $OUT/lone_factors.jsonl 2>&1
