mkdir -p gpurun_out/r2j
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2j/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r2j/smoke.log
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > gpurun_out/r2j/pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2j/pytest.log
timeout 900 python bench.py > gpurun_out/r2j/bench.json 2> gpurun_out/r2j/bench.err; echo bench_rc=$? >> gpurun_out/r2j/bench.err
