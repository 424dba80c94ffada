mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2c/pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2c/pytest.log
AB_N=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 170 -c 1 -o gpurun_out/r2c/chain python tools/ttft_ab.py ncu > gpurun_out/r2c/ncu.log 2>&1
