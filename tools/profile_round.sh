#!/bin/bash
# One GPU session of evidence for profiles/: bench line, reference arm, ncu launch list of
# one cached 7B request, and full ncu captures of the top kernels (GEMM, attention, assembly).
# Usage (under gpurun): bash tools/profile_round.sh <tag>
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
nproc > $OUT/host.txt; grep -m1 "model name" /proc/cpuinfo >> $OUT/host.txt; free -g >> $OUT/host.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# launch list of one full-depth cached request (after warm-up requests)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/launches.csv python tools/prof_step.py > $OUT/launches.log 2>&1
# full captures of the top kernels (2 layers keep the replay short).  Launch order: the
# module precompute (4096-token prefill: per-GEMM k_gemm_2sm, one k_attn_prefill per layer),
# the warm-up request, then the measured request -- at 2 layers each request is ONE chain launch
# ([LN1, QKV0, ATTN0, O, W1, W2, QKV1, ATTN1, O, W1, W2, unembed]); skip counts below.
cap() {  # kernel-regex skip count
  PROF_LAYERS=2 PROF_WARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 \
    -o $OUT/full_$1 python tools/prof_step.py > $OUT/full_$1.log 2>&1
}
cap k_chain 1 1
cap k_attn_prefill 0 1
PROF_ZC=0 cap k_assemble 1 1  # single requests read modules in place; the copy path is measured with it off
ls -la $OUT
