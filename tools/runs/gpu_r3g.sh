#!/bin/bash
# evidence pass after the k_attn_tc (batched / suffix attention) rework
OUT=gpurun_out/r3g
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
bash tools/profile_round.sh r3g
AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 2 > $OUT/chain_tl.txt 2>&1
