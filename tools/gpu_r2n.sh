mkdir -p gpurun_out/r2n
rm -f gpurun_out/r2n/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2n/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_serve.py -x -q -p no:cacheprovider > gpurun_out/r2n/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2n/pytest.log
for w in 0 1; do
  echo "== dsm=$w" >> gpurun_out/r2n/ab.txt
  PCB_CHAIN_DSM=$w AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 2 >> gpurun_out/r2n/ab.txt 2>&1
done
