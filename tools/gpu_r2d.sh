mkdir -p gpurun_out/r2d
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2d/pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2d/pytest.log
timeout 300 python tools/ttft_ab.py new >> gpurun_out/r2d/ab.log 2>&1
