mkdir -p gpurun_out/exp1
for v in 1 0; do
  PCB_GEMM_COLOC=$v timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-slow > gpurun_out/exp1/bench_coloc$v.json 2> gpurun_out/exp1/bench_coloc$v.err
done
for sp in 2 4 8; do
  PCB_ATTN_SPLITS=$sp timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-slow > gpurun_out/exp1/bench_split$sp.json 2> gpurun_out/exp1/bench_split$sp.err
done
PCB_PDL_MASK=127 timeout 300 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-slow > gpurun_out/exp1/bench_pdlall.json 2> gpurun_out/exp1/bench_pdlall.err
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/exp1/pytest.log 2>&1
