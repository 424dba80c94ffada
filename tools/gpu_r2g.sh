mkdir -p gpurun_out/r2g
for mb in 16 32 64; do timeout 300 python tools/c4_profile.py $mb >> gpurun_out/r2g/c4prof.log 2>&1; done
for mb in 16 32 16 32 64; do C4_N=256 timeout 300 python tools/c4_timing.py $mb 2>&1 | head -3 >> gpurun_out/r2g/c4tim.log; done
