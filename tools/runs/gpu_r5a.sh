#!/bin/bash
# evidence pass at the start of the last session (HEAD after the launch-boundary probes): smoke, -m gpu, bench + reference arm + launch list + ncu captures, timelines
OUT=gpurun_out/r5a
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
bash tools/profile_round.sh r5a
AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 2 > $OUT/chain_tl.txt 2>&1
AB_CACHED=16384 AB_UNC=128 AB_MODS=3 AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c3.txt 2>&1
