mkdir -p gpurun_out/r2e
timeout 600 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "multiproc or pcst or peer" > gpurun_out/r2e/pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2e/pytest.log
