#!/bin/bash
# final-state check with the cooperative chain launch on by default:
# smoke, -m gpu, both bench arms as the driver runs them
OUT=gpurun_out/r5e
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
