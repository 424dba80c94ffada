#!/bin/bash
# ncu full captures for the multi-layer chain + paired prefill attention (profile_round's cap list)
OUT=gpurun_out/r2z
mkdir -p $OUT
cap() {
  PROF_LAYERS=2 PROF_WARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 \
    -o $OUT/full_$1 python tools/prof_step.py > $OUT/full_$1.log 2>&1
}
rm -f $OUT/full_k_chain* $OUT/full_k_attn*
cap k_chain 1 1
cap k_attn_prefill 0 1
