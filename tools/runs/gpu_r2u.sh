#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over smoke(): one fp32 and one bf16
# cached serve of the tiny model (SIMT, tcgen05 GEMM, attention and chain kernels)
OUT=gpurun_out/r2u
mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -c "import __graft_entry__ as g; g.smoke()" > $OUT/$tool.log 2>&1
  echo "rc=$?" >> $OUT/$tool.log
done
# PDL for the attention class (PCB_PDL_MASK bit 2) re-tested on the standalone-attention path
PCB_PDL_MASK=127 timeout 600 python -m pytest tests/test_gpu_kernels.py -k "cached_serve_equals_oracle or tc_path_vs_simt or paired" -x -q -p no:cacheprovider > $OUT/pdl_attn.log 2>&1; echo rc=$? >> $OUT/pdl_attn.log
