mkdir -p gpurun_out/r2m
rm -f gpurun_out/r2m/ab.txt
for w in 0 1; do
  echo "== warm=$w" >> gpurun_out/r2m/ab.txt
  PCB_CHAIN_WARM=$w AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 2 >> gpurun_out/r2m/ab.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_serve.py -x -q -p no:cacheprovider > gpurun_out/r2m/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2m/pytest.log
