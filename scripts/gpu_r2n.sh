#!/bin/bash
# Session n: the bench's default line (e2e + cpu_baseline + parity record) after the parity-record
# fix, the two-rank GPU tests (incl. reduce-to-owner), then the Ozaki digit-count experiment.
OUT=gpurun_out/r2n; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_ozaki.py -q -rA > $OUT/pytest_dist.log 2>&1; echo "rc=$?" >> $OUT/pytest_dist.log
timeout 900 python bench.py > $OUT/bench_r50_default.json 2> $OUT/bench_r50_default.err
TAG=r2n/ozd bash scripts/gpu_ozdigits.sh
