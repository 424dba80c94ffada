mkdir -p gpurun_out/r2b
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2b/pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2b/pytest.log
for i in 1 2; do
PCB_LIB_PATH=ablib/base/libpcb200.so timeout 300 python tools/ttft_ab.py base >> gpurun_out/r2b/ab.log 2>&1
timeout 300 python tools/ttft_ab.py new >> gpurun_out/r2b/ab.log 2>&1
done
timeout 600 python tools/chain_ab.py 2 > gpurun_out/r2b/chain_tl.txt 2>&1
