#!/bin/bash
# Workspace-poison tests + compute-sanitizer initcheck of the two-stage d = 1041 case.
OUT=gpurun_out/${TAG:-poison}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ws_poison.py -q -rA > $OUT/pytest_poison.log 2>&1; echo "rc=$?" >> $OUT/pytest_poison.log
timeout 900 compute-sanitizer --tool initcheck --print-limit 30 python -m pytest tests/test_gpu_ws_poison.py -q -x -k "1041-300-12" > $OUT/initcheck_1041.log 2>&1; echo "rc=$?" >> $OUT/initcheck_1041.log
