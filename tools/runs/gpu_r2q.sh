#!/bin/bash
# chain timeline (current build), GEMM sweep with clocks, ncu full captures of k_gemm_2sm
OUT=gpurun_out/r2q
mkdir -p $OUT
AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 2 > $OUT/chain_tl.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw --format=csv -lms 200 > $OUT/kbench_clocks.csv &
SMI=$!
timeout 300 python tools/kbench.py > $OUT/kbench.txt 2>&1
kill $SMI 2>/dev/null
for shp in "4160 12288 4096" "4160 16384 4096" "4160 4096 16384" "2048 12288 4096" "4096 16384 4096"; do
  tag=$(echo $shp | tr ' ' '_')
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 1 \
    -o $OUT/gemm_$tag python tools/gemm_ncu.py $shp > $OUT/gemm_$tag.log 2>&1
done
ls -la $OUT
