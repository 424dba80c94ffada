"""Config 4 micro-batch timeline: device time per micro-batch of serve_batch and each
micro-batch's assembly / prefill / TTFT split.
  C4_N=256 python tools/c4_timing.py [micro_batch]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2311_04934_b200 as pcb
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
m = pcb.Model(bench.CFG_7B, dtype=pcb.BF16)
schema_text, prompts, _ = bench.workload_c4(64, 256, 256, 8, 64)
schema = pcb.Schema.parse(schema_text)
store = pcb.ModuleStore(m)
store.encode_schema(schema)
ps = [pcb.Prompt.parse(p) for p in prompts[: int(os.environ.get("C4_N", 8 * mb))]]
pcb.serve_batch(store, schema, ps[: 2 * mb], micro_batch=mb)
m.sync()
m.timer_start(); t0 = time.perf_counter()
stop = []
res = pcb.serve_batch(store, schema, ps, micro_batch=mb, after=lambda: stop.append(m.timer_stop()))
dev = stop[0]; wall = (time.perf_counter() - t0) * 1e3
nb = len(ps) // mb
print(f"mb {mb}: device {dev/nb:.2f} ms/micro-batch, wall {wall/nb:.2f}")
for k in range(nb):
    t = res[k * mb].timings
    print(f"  mb{k}: asm {t['assemble_us']/1e3:.2f} prefill {t['prefill_device_us']/1e3:.2f} ttft {t['ttft_us']/1e3:.2f} parse {t.get('parse_us',0)/1e3:.2f}")
