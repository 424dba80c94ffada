"""Summarise a gpurun_out/<tag>/ profiling session (tools/profile_round.sh) into profiles/<tag>_*.

Writes:
  profiles/<tag>_launches.csv   per-launch device time + DRAM bytes of one cached 7B request (ncu)
  profiles/<tag>_summary.md     kernel-class shares, ncu --set full metrics of the top kernels,
                                the bench line and the reference-arm line
  profiles/<tag>_traffic.json   DRAM bytes per step of the GEMM class (read by bench.py)
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: i for i, k in enumerate(hdr)}
    k = collections.defaultdict(dict)
    for r in rows[start + 1:]:
        kid = int(r[ix["ID"]])
        k[kid]["name"] = r[ix["Kernel Name"]]
        k[kid][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    return k


def short(name):
    n = name.split("(")[0].replace("void ", "")
    return n.split("::")[-1].split("<")[0] if "::" in n else n.split("<")[0]


def ncu_metrics(rep, want):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for w in want:
            if w in hdr:
                u = units[hdr.index(w)]
                d[w] = r[hdr.index(w)] + (f" {u}" if u and u not in ("%",) else "")
        res.append(d)
    return res


def main(tag):
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    k = read_launches(os.path.join(src, "launches.csv"))
    ids = sorted(k)
    # the measured request: every launch after the previous request's argmax up to its own
    # (it starts with the assembly copy, or -- zero-copy -- with the embedding)
    args = [i for i in ids if "k_argmax" in k[i]["name"]]
    last_arg = args[-1]
    prev_arg = args[-2] if len(args) > 1 else -1
    step = [i for i in ids if prev_arg < i <= last_arg]
    first_asm = step[0]
    with open(os.path.join(dst, f"{tag}_launches.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["launch", "kernel", "gpu_time_us", "dram_read_bytes", "dram_write_bytes"])
        for i in step:
            w.writerow([i - first_asm, short(k[i]["name"]), k[i]["gpu__time_duration.sum"] / 1e3,
                        int(k[i].get("dram__bytes_read.sum", 0)), int(k[i].get("dram__bytes_write.sum", 0))])
    tot = sum(k[i]["gpu__time_duration.sum"] for i in step)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i in step:
        a = agg[short(k[i]["name"])]
        a[0] += 1
        a[1] += k[i]["gpu__time_duration.sum"]
        a[2] += k[i].get("dram__bytes_read.sum", 0) + k[i].get("dram__bytes_write.sum", 0)
    gemm_kernels = ("k_chain", "k_gemm_sk")  # the GEMM class: persistent chains (+ any per-GEMM launches)
    gemm_traffic = sum(agg[g][2] for g in gemm_kernels if g in agg)
    with open(os.path.join(dst, f"{tag}_traffic.json"), "w") as f:
        json.dump({"gemm_dram_bytes_per_step": gemm_traffic,
                   "gemm_launches_per_step": sum(agg[g][0] for g in gemm_kernels if g in agg),
                   "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one cached request "
                             f"(profiles/{tag}_launches.csv)"}, f, indent=1)

    lines = [f"# Profile {tag}: one cached Llama-2-7B-shape request (4096 cached + 64 uncached)", ""]
    for fn in ("gpu.txt", "host.txt"):
        p = os.path.join(src, fn)
        if os.path.exists(p):
            lines += ["```", open(p).read().strip(), "```", ""]
    lines += ["## Launch list (ncu `gpu__time_duration.sum`, cold caches, serialised)", "",
              f"{len(step)} launches, {tot / 1e6:.3f} ms summed device time.", "",
              "| kernel | launches | time (us) | share | DRAM bytes | DRAM GB/s |", "|---|---|---|---|---|---|"]
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {n} | {c} | {t / 1e3:.1f} | {t / tot * 100:.1f}% | {b / 1e9:.3f} G | {b / t:.0f} |")
    want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    for kern in ("k_chain", "k_gemm_sk", "k_attn_tc", "k_attn_prefill", "k_assemble"):
        rep = os.path.join(src, f"full_{kern}.ncu-rep")
        if not os.path.exists(rep):
            continue
        ms = ncu_metrics(rep, want)
        lines += ["", f"## ncu --set full: {kern} ({len(ms)} launch(es) captured)", ""]
        if ms:
            cols = [c for c in want if c in ms[0] and c != "Kernel Name"]
            lines.append("| " + " | ".join(cols) + " |")
            lines.append("|" + "---|" * len(cols))
            for m in ms:
                lines.append("| " + " | ".join(m.get(c, "") for c in cols) + " |")
    for fn in ("bench.json", "bench_ref.json"):
        p = os.path.join(src, fn)
        if os.path.exists(p) and os.path.getsize(p):
            lines += ["", f"## {fn}", "", "```json", open(p).read().strip(), "```"]
    with open(os.path.join(dst, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
