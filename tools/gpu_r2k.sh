# round-2 evidence: bench + reference arm + launch list + ncu full captures (chain, prefill attention,
# assembly), chain timeline, k_gemm_2sm captures at prefill / config-4 sizes
bash tools/profile_round.sh r2a
mkdir -p gpurun_out/r2a
AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > gpurun_out/r2a/chain_tl.txt 2>&1
timeout 300 python tools/kbench.py > gpurun_out/r2a/kbench.log 2>&1
cat > /tmp/gk.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import kbench
for M in (4160, 4096, 2048):
    kbench.bench("gemm", M, 16384, 4096, iters=2)
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_2sm -s 2 -c 3 -o gpurun_out/r2a/full_k_gemm_2sm python /tmp/gk.py > gpurun_out/r2a/full_gemm.log 2>&1
