#!/bin/bash
# End-of-session evidence: full suite + smoke + bench lines + launch list + ncu captures.
TAG=${TAG:-final}
OUT=gpurun_out/$TAG; mkdir -p $OUT
TAG=$TAG CONFIGS="mlp r32 r101" bash scripts/gpu_full.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_r50.csv \
  python bench.py --config r50 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_list.log 2>&1
TAG=$TAG SPECS="trd_panel:5:1 gemm64_direct:40:1 syrk_tc_planes8:0:1 gemm_tc_planes:2:1" bash scripts/gpu_ncu.sh
python scripts/eig_scaling.py --config r50 > $OUT/eig_scaling_r50.jsonl 2>&1
for v in inverse factored; do   # C4: explicit-inverse (Eqs. 11-12) and factored-damping variants
  timeout 900 python bench.py --config r50 --variant $v --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r50_$v.json 2> $OUT/bench_r50_$v.err
done
