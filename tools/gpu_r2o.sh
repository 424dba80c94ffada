mkdir -p gpurun_out/r2o
PROF_LAYERS=2 PROF_WARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 3 -c 2 -o gpurun_out/r2o/full_k_chain python tools/prof_step.py > gpurun_out/r2o/ncu.log 2>&1
