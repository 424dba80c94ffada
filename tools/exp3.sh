mkdir -p gpurun_out/exp3
timeout 300 python __graft_entry__.py > gpurun_out/exp3/smoke.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/exp3/pytest.log 2>&1
for pf in 0 24 64; do
  PCB_CHAIN_PF=$pf timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-slow > gpurun_out/exp3/bench_pf$pf.json 2> gpurun_out/exp3/bench_pf$pf.err
done
PCB_CHAIN=0 timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-slow > gpurun_out/exp3/bench_nochain.json 2> gpurun_out/exp3/bench_nochain.err
