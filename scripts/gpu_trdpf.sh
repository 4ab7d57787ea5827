#!/bin/bash
# trd_panel L2-prefetch experiment: for each threshold (MB of lower-triangle working set above which a
# launch prefetches each warp's next symv unit into L2; 100000 = never, 0 = always) build, run the
# eigen GPU tests once, one r50 bench line and the lone-factor times.  Outputs under gpurun_out/$TAG.
TAG=${TAG:-trdpf}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for T in ${THRESH:-100000 96 0}; do
  export KFAC_NVCC_EXTRA="-DKFAC_TRD_L2PF_MB=$T $EXTRA"
  python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$T.log 2>&1
  if [ "$T" = "96" ]; then
    timeout 900 python -m pytest tests/test_gpu_eigen_trd.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x > $OUT/pytest_$T.log 2>&1; echo "rc=$?" >> $OUT/pytest_$T.log
  fi
  timeout 600 python bench.py --config r50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r50_$T.json 2> $OUT/bench_r50_$T.err
  timeout 300 python scripts/sbr_time.py 2305 4609 > $OUT/lone_$T.jsonl 2>&1
done
unset KFAC_NVCC_EXTRA
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_default.log 2>&1
