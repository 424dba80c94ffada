#!/bin/bash
# verification after cleanups: smoke, -m gpu, bench line
OUT=gpurun_out/r3l
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
