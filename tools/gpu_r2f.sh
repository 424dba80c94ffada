mkdir -p gpurun_out/r2f
cd gpurun_out/r2f
PCB_ATTN_DBG=1 timeout 300 python ../../tools/kbench.py > kbench_dbg.log 2>&1
timeout 300 python ../../tools/kbench.py > kbench.log 2>&1
cat > /tmp/gk.py <<'PY'
import sys; sys.path.insert(0, "../../tools"); sys.path.insert(0, "../..")
import kbench
for M in (4160, 2048, 256):
    kbench.bench("gemm", M, 16384, 4096, iters=2)
kbench.bench("attn", 4160, 0, 32, iters=2)
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_2sm|k_attn_tc" -c 8 -o gemm_attn python /tmp/gk.py > ncu.log 2>&1
