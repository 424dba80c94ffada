#!/bin/bash
# LayerNorm folded into the CTA-pair GEMMs: parity, config-4 A/B, full prefill / precompute
OUT=gpurun_out/r3r
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2 3; do for v in 0 1; do
  echo "== fold=$v" >> $OUT/c4.txt
  PCB_LN_FOLD_BIG=$v C4_N=256 timeout 600 python tools/c4_timing.py 64 2>&1 | head -1 >> $OUT/c4.txt
done; done
for v in 0 1; do
PCB_LN_FOLD_BIG=$v python - >> $OUT/prefill.txt 2>&1 <<'PY'
import os, sys, time
sys.path.insert(0, ".")
import bench, paper_2311_04934_b200 as pcb
m = pcb.Model(bench.CFG_7B, dtype=pcb.BF16)
schema_text, prompts = bench.workload(4096, 64, 1)
s = pcb.Schema.parse(schema_text)
st = pcb.ModuleStore(m); st.encode_schema(s); m.sync()
t0 = time.perf_counter(); st2 = pcb.ModuleStore(m); st2.encode_schema(s); m.sync(); pre = (time.perf_counter() - t0) * 1e3
fp = [pcb.serve(st2, s, prompts[0], max_new_tokens=1, use_cache=False).timings["ttft_us"] / 1e3 for _ in range(4)][1:]
print(f"fold_big={os.environ['PCB_LN_FOLD_BIG']}: precompute {pre:.1f} ms, full prefill {min(fp):.1f} ms")
PY
done
