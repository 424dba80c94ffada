mkdir -p gpurun_out/exp2
timeout 300 python __graft_entry__.py > gpurun_out/exp2/smoke.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/exp2/pytest.log 2>&1
for v in 1 0; do
  PCB_CHAIN=$v timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-slow > gpurun_out/exp2/bench_chain$v.json 2> gpurun_out/exp2/bench_chain$v.err
done
