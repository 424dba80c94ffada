#!/bin/bash
# compute-sanitizer over the hd128 workload after the last-session kernel changes (LDS/STS pointers, inline watchdogs, lean 128-token epilogue)
OUT=gpurun_out/r4n
mkdir -p $OUT
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 --error-exitcode 9 python tools/sanitize_hd128.py > $OUT/san_$tool.log 2>&1
  echo "rc=$?" >> $OUT/san_$tool.log
done
