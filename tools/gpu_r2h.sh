mkdir -p gpurun_out/r2h
PCB_BATCH_TRACE=1 C4_N=256 timeout 300 python tools/c4_timing.py 64 > gpurun_out/r2h/c4_64.log 2>&1
PCB_BATCH_TRACE=1 C4_N=256 timeout 300 python tools/c4_timing.py 32 > gpurun_out/r2h/c4_32.log 2>&1
