"""A/B of few-token forward variants inside ONE process (box-to-box noise is ~10%), plus a
timeline of the persistent chain kernel for one 7B-shape cached request.

  python tools/chain_ab.py [rounds]
Variants are model options (set_option): chain on/off.
"""
import ctypes as C
import os
import statistics
import sys

os.environ.setdefault("PCB_CHAIN_PROBE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import numpy as np  # noqa: E402

import paper_2311_04934_b200 as pcb  # noqa: E402

L = pcb.lib()
L.pcb_debug_chain_probe.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_void_p]
MAXL = 64
KMAX = 48  # kern::kChainMaxPhases
times = np.zeros((MAXL, KMAX, 160, 16), np.uint64)
phases = np.zeros(MAXL, np.int32)


def dump():
    n = C.c_int()
    rc = L.pcb_debug_chain_probe(times.ctypes.data, MAXL, C.byref(n), phases.ctypes.data)
    assert rc == 0, L.pcb_last_error()
    return n.value


VARIANTS = [
    ("per-GEMM kernels", {"chain": 0, "zero_copy": 0}),
    ("chain", {"chain": 1, "ln_fold": 1, "chain_attn": 0, "zero_copy": 0}),
    ("chain+attn", {"chain": 1, "ln_fold": 1, "chain_attn": 1, "zero_copy": 0}),
    ("zero-copy", {"chain": 1, "ln_fold": 1, "chain_attn": 1, "zero_copy": 1}),
    ("chain, LN phases", {"chain": 1, "ln_fold": 0, "chain_attn": 0, "zero_copy": 0}),

]
if os.environ.get("AB_VARIANTS"):
    VARIANTS = [v for v in VARIANTS if v[0] in os.environ["AB_VARIANTS"].split(",")]

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 5
layers = int(os.environ.get("PROF_LAYERS", "32"))
cfg = dict(bench.CFG_7B, n_layers=layers, max_position=32768)
schema_text, prompts = bench.workload(int(os.environ.get("AB_CACHED", "4096")), int(os.environ.get("AB_UNC", "64")),
                                     int(os.environ.get("AB_MODS", "1")))  # configs[2]: 16384 128 3
m = pcb.Model(cfg, dtype=pcb.BF16)
s = pcb.Schema.parse(schema_text)
st = pcb.ModuleStore(m)
st.encode_schema(s)
parsed = [pcb.Prompt.parse(p) for p in prompts]
res = {name: [] for name, _ in VARIANTS}
for r in range(rounds):
    for name, opts in VARIANTS:
        for k, v in opts.items():
            if k.startswith("env:"):
                os.environ[k[4:]] = str(v)
            else:
                m.set_option(k, v)
        pcb.serve(st, s, parsed[0], max_new_tokens=1)  # settle
        for i in range(3):
            rr = pcb.serve(st, s, parsed[(i + 1) % len(parsed)], max_new_tokens=1)
            res[name].append(rr.timings["ttft_us"] / 1e3)
        dump()
print("TTFT ms (median / min over", rounds * 3, "requests)")
for name, v in res.items():
    print(f"  {name:18s} {statistics.median(v):7.3f} {min(v):7.3f}")

# ---- chain timeline of one request ----
m.set_option("chain", 1)
m.set_option("ln_fold", int(os.environ.get("TL_FOLD", "1")))
m.set_option("chain_attn", int(os.environ.get("TL_ATTN", "1")))
m.set_option("zero_copy", int(os.environ.get("TL_ZC", "1")))
pcb.serve(st, s, parsed[0], max_new_tokens=1)
m.sync()
dump()
pcb.serve(st, s, parsed[1], max_new_tokens=1)
n = dump()
names6 = ["O", "LN2", "W1", "W2", "LN1", "QKV"] if os.environ.get("TL_FOLD", "1") == "0" else ["O", "W1", "W2", "QKV"]
print(f"chain launches {n}")
agg = {}
prev_end = None
for i in range(n):
    npn = int(phases[i])
    t = times[i, :npn, :148].astype(np.int64)  # [ph][cta][ev]
    kinds = times[i, :npn, 159, 15].astype(np.int64) - 1  # 0 GEMM, 1 LN, 2 ATTN
    names, after = [], None
    for kd in kinds:
        if kd == 1:
            names.append("LN1")
            after = 3
        elif kd == 2:
            names.append("ATTN")
            after = 0
        else:
            names.append(["O", "W1", "W2", "QKV"][after] if after is not None and after < 4 else "GEMM")
            after = (after + 1) if after is not None else None
    for ph in range(npn):
        ev = t[ph]
        act = ev[:, 2] > 0  # CTAs of the grid (a cluster launch uses fewer than 148)
        done = ev[act, 2]
        start_x = ev[:, 0]
        row = {}
        if ph > 0:
            prev_done_max = t[ph - 1][:, 2].max()
            row["barrier"] = (np.median(start_x[start_x > 0]) - prev_done_max) / 1e3 if (start_x > 0).any() else None
        row["done_spread"] = (done.max() - done.min()) / 1e3
        if (start_x > 0).any():
            mma_end = ev[:, 1]
            ok = (start_x > 0) & (mma_end > 0)
            row["stream"] = np.median((mma_end - start_x)[ok]) / 1e3
            row["epi_tail"] = np.median((ev[:, 2] - mma_end)[ok]) / 1e3
            row["w_lead"] = np.median((start_x - ev[:, 3])[ok]) / 1e3  # >0: weights issued before barrier passed
        if (start_x > 0).any():
            okk = (ev[:, 6] > 0) & (ev[:, 7] > 0)
            row["poll"] = np.median((ev[:, 7] - ev[:, 6])[okk]) / 1e3
            row["proxyfence"] = np.median((ev[:, 0] - ev[:, 7])[okk]) / 1e3
            row["pass_minus_lastdone"] = (np.median(ev[:, 7][okk]) - (t[ph - 1][:, 2].max() if ph > 0 else 0)) / 1e3 if ph > 0 else None
            ok4 = (ev[:, 4] > 0) & (ev[:, 1] > 0)
            row["accwait_after_mma"] = np.median((ev[:, 4] - ev[:, 1])[ok4]) / 1e3
            ok9 = (ev[:, 9] > 0) & (ev[:, 4] > 0) & (ev[:, 10] > 0) & (ev[:, 11] == 0)
            if ok9.any():  # S == 1 epilogue: chunk loop, staged-store copy, tail
                row["s1_loop"] = np.median((ev[:, 9] - ev[:, 4])[ok9]) / 1e3
                row["s1_copy"] = np.median((ev[:, 10] - ev[:, 9])[ok9]) / 1e3
                row["s1_tail"] = np.median((ev[:, 5] - ev[:, 10])[ok9]) / 1e3
                okc = ok9 & (ev[:, 15] > 0)
                if okc.any():  # first two chunks: TMEM load / values + smem staging
                    row["c0_ld"] = np.median((ev[:, 12] - ev[:, 4])[okc]) / 1e3
                    row["c0_val"] = np.median((ev[:, 13] - ev[:, 12])[okc]) / 1e3
                    row["c1_ld"] = np.median((ev[:, 14] - ev[:, 13])[okc]) / 1e3
                    row["c1_val"] = np.median((ev[:, 15] - ev[:, 14])[okc]) / 1e3
            ok5 = (ev[:, 5] > 0) & (ev[:, 4] > 0)
            if ok5.any():
                row["flagwait"] = np.median((ev[:, 5] - ev[:, 4])[ok5]) / 1e3
                row["owner_epi"] = np.median((ev[:, 2] - ev[:, 5])[ok5]) / 1e3
                ok8 = ok5 & (ev[:, 9] > 0) & (ev[:, 11] > 0)
                if ok8.any():
                    row["o_partials"] = np.median((ev[:, 9] - ev[:, 5])[ok8]) / 1e3
                    row["o_epi"] = np.median((ev[:, 10] - ev[:, 9])[ok8]) / 1e3
                    row["o_stats"] = np.median((ev[:, 11] - ev[:, 10])[ok8]) / 1e3
                    row["o_after"] = np.median((ev[:, 2] - ev[:, 11])[ok8]) / 1e3
        first_done = t[0][:, 2]
        row["phase_span"] = (done.max() - (t[ph - 1][:, 2].max() if ph > 0 else first_done[first_done > 0].min())) / 1e3
        agg.setdefault(names[ph], []).append(row)
    first = t[0][:, 0]
    first = first[first > 0]
    if prev_end is not None and len(first):
        agg.setdefault(("gap", "attention+launch"), []).append({"gap": (first.min() - prev_end) / 1e3})
    prev_end = t[npn - 1][:, 2].max()
# attention-phase cycle accounting (raw clock64 counts in slots 12-15 of phase 0)
cyc = []
for i in range(n):
    for ph in range(int(phases[i])):
        if times[i, ph, 159, 15] != 3:  # attention phases only
            continue
        ev = times[i, ph, :128].astype(np.int64)
        ok = ev[:, 12] > 0
        if ok.any():
            cyc.append([np.median(ev[ok, k]) for k in (12, 13, 14, 15, 6, 7)])
if cyc:
    c = np.median(np.array(cyc), axis=0)
    print(f"ATTN cycles (median CTA, median chain): softmax loop {c[0]:.0f}, of which waiting for S {c[1]:.0f}; "
          f"MMA waiting for K/V {c[2]:.0f}, for P {c[3]:.0f}; output/park loop {c[4]:.0f}, split merge {c[5]:.0f}")
# launch boundaries (probe slot of phase KMAX - 1): previous chain's last exit -> this chain's
# first CTA entry -> prologue done -> past the PDL wait -> first phase-0 event
gaps = []
for i in range(1, n):
    e_prev = times[i - 1, KMAX - 1, :160, 3].astype(np.int64)
    e = times[i, KMAX - 1, :160].astype(np.int64)
    ok = e[:, 0] > 0
    if not ok.any() or not (e_prev > 0).any():
        continue
    t_exit = e_prev[e_prev > 0].max()
    ph0 = times[i, 0, :160, 0].astype(np.int64)
    ph0 = ph0[ph0 > 0]
    gaps.append([(e[ok, 0].min() - t_exit) / 1e3, (e[ok, 0].max() - t_exit) / 1e3, (e[ok, 1].max() - t_exit) / 1e3,
                 (e[ok, 2][e[ok, 2] > 0].max() - t_exit) / 1e3 if (e[ok, 2] > 0).any() else float("nan"),
                 (ph0.min() - t_exit) / 1e3 if len(ph0) else float("nan")])
if gaps:
    g = np.median(np.array(gaps), axis=0)
    print(f"launch boundary (median of {len(gaps)}), us after the previous chain's last exit: first entry {g[0]:.1f}, "
          f"last entry {g[1]:.1f}, prologue done {g[2]:.1f}, past PDL wait {g[3]:.1f}, first phase-0 event {g[4]:.1f}")
print("per phase (median over chains), us")
for key, rows in agg.items():
    keys = sorted({k for r_ in rows for k in r_})
    out = []
    for k in keys:
        vals = [r_[k] for r_ in rows if r_.get(k) is not None]
        if vals:
            out.append(f"{k} {statistics.median(vals):6.1f}")
    print(f"  {str(key):28s} x{len(rows):3d}  " + "  ".join(out))

# ---- attention phase: per-CTA event distribution (us from the earliest phase start) ----
if os.environ.get("TL_ATTN", "1") != "0":
    rows = []
    for i in range(n):
        for ph in range(int(phases[i])):
            if times[i, ph, 159, 15] != 3:
                continue
            ev = times[i, ph, :128].astype(np.int64)
            t0 = ev[:, 0][ev[:, 0] > 0].min()
            rows.append([(ev[:, k] - t0) / 1e3 for k in (0, 1, 9, 10, 4, 8, 5, 11, 2)])
    if rows:
        a = np.array(rows)  # [chain][event][cta]
        print("ATTN per-CTA events (median over chains of the percentile), us: start / last PV / dup merged / parked / a_done / released / flags / merged / done")
        for q in (0, 50, 90, 100):
            print(f"  p{q:3d}  " + "  ".join(f"{np.median(np.percentile(a[:, k, :], q, axis=1)):6.1f}" for k in range(9)))
        # is the straggler split a fixed one (last split holds the diagonal block)?
        lastpv = np.median(a[:, 1, :], axis=0).reshape(-1, 4)
        print("  last PV by split (median over heads):", np.round(np.median(lastpv, axis=0), 1))
        print("  last PV by head (median over splits):", np.round(np.median(lastpv, axis=1), 1))
