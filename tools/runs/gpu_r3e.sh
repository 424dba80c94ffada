#!/bin/bash
# k_attn_tc with P in TMEM and three score buffers: parity (all attention users), config-4 breakdown, kbench
OUT=gpurun_out/r3e
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 600 python tools/c4_profile.py 64 > $OUT/c4prof64.txt 2>&1
timeout 300 python tools/kbench.py > $OUT/kbench.txt 2>&1
