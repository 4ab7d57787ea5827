#!/bin/bash
# Ozaki digit-count experiment: for each S in $DIGITS build libkfac with -DKFAC_OZ_DIGITS=S, run the
# whole GPU suite and one r50 bench line.  Outputs under gpurun_out/$TAG.
TAG=${TAG:-ozd}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for S in ${DIGITS:-5 4}; do
  export KFAC_NVCC_EXTRA="-DKFAC_OZ_DIGITS=$S"
  python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$S.log 2>&1
  timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_$S.log 2>&1; echo "rc=$?" >> $OUT/pytest_$S.log
  timeout 600 python bench.py --config r50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r50_$S.json 2> $OUT/bench_r50_$S.err
done
unset KFAC_NVCC_EXTRA
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_default.log 2>&1
