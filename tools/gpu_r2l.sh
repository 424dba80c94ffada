# A/B: dry epilogue pass (instruction-cache warm-up) in the chain's S=1 phases
mkdir -p gpurun_out/r2l
for r in 1 2; do
for w in 0 1; do
  echo "== warm=$w round $r" >> gpurun_out/r2l/ab.txt
  PCB_CHAIN_WARM=$w AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 2 >> gpurun_out/r2l/ab.txt 2>&1
done
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/r2l/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2l/pytest.log
