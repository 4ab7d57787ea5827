#!/bin/bash
# Quick GPU check: build, selected gpu tests, one bench line per config.  TAG, TESTS, BENCH_CONFIGS.
OUT=gpurun_out/${TAG:-q}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest ${TESTS:-tests} -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for c in ${BENCH_CONFIGS:-r50}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
