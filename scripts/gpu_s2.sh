OUT=gpurun_out/s2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for dr in 1 2 4 8; do
  KFAC_TC_DRAIN_SYRK=$dr KFAC_TC_DRAIN_GEMM=$dr timeout 600 python bench.py --config r50 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/bench_d$dr.json 2> $OUT/bench_d$dr.err
done
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_d1.log 2>&1
KFAC_TC_DRAIN_SYRK=4 KFAC_TC_DRAIN_GEMM=4 timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_d4.log 2>&1
