mkdir -p gpurun_out/dbg4
for m in 59 107 115 121 91 122 123; do
  PCB_PDL_MASK=$m timeout 100 python -m pytest tests/test_gpu_kernels.py -x -q -k "oracle_7b or deterministic" > gpurun_out/dbg4/mask$m.log 2>&1
  echo "mask $m rc $?" >> gpurun_out/dbg4/summary.txt
done
