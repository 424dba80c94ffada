mkdir -p gpurun_out/r2i
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2i/pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2i/pytest.log
for mb in 32 64; do
C4_N=256 timeout 300 python tools/c4_timing.py $mb 2>&1 | head -1 >> gpurun_out/r2i/c4.log
PCB_ATTN_NODUP=1 C4_N=256 timeout 300 python tools/c4_timing.py $mb 2>&1 | head -1 | sed 's/^/nodup /' >> gpurun_out/r2i/c4.log
done
timeout 300 python tools/c4_profile.py 32 >> gpurun_out/r2i/c4.log 2>&1
