"""Summarise an official round measurement (scripts/gpu_official.sh TAG) into markdown:
launch-list shares (tmc kernels only, torch/cuBLAS harness kernels grouped) and the full-capture
metrics of the captured tc_* kernels.  Usage: python scripts/ncu_summary.py TAG > profiles/<file>.md"""
import collections, csv, json, subprocess, sys

tag = sys.argv[1]
out = []
rows = list(csv.reader(open(f"gpurun_out/launches_{tag}.csv")))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        ours = any(k in name for k in ("tc::", "simt::", "tc_", "pass_kernel", "hbuild", "unary_", "final_", "xmsg", "hroot"))
        key = name.split("(")[0] if ours else "(harness / torch / cuBLAS kernels)"
        v = float(d["Metric Value"].replace(",", ""))
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += v
tot = sum(v[1] for v in agg.values())
out.append(f"## Launch list ({tag}): share of GPU time per kernel\n")
out.append("| share | launches | us/launch | kernel |\n|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f"| {100 * t / tot:.2f}% | {n} | {t / n / 1e3:.1f} | `{k[:110]}` |")
raw = subprocess.run(["ncu", "-i", f"gpurun_out/prof_full_{tag}.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
R = list(csv.reader(raw.splitlines()))
if len(R) > 2:
    h, u = R[0], R[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__block_size"]
    idx = {w: h.index(w) for w in want if w in h}
    kn = h.index("Kernel Name")
    out.append(f"\n## Full capture ({tag})\n")
    out.append("| metric | unit | " + " | ".join(f"launch {i + 1}: `{r[kn][:40]}`" for i, r in enumerate(R[2:])) + " |")
    out.append("|---|---|" + "---|" * (len(R) - 2))
    for w, i in idx.items():
        out.append(f"| `{w}` | {u[i]} | " + " | ".join(r[i] for r in R[2:]) + " |")
    tr = []
    for r in R[2:]:
        rd, wr = float(r[idx["dram__bytes_read.sum"]].replace(",", "")), float(r[idx["dram__bytes_write.sum"]].replace(",", ""))
        sc = lambda unit: {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(unit, 1)
        tr.append(rd * sc(u[idx["dram__bytes_read.sum"]]) + wr * sc(u[idx["dram__bytes_write.sum"]]))
    out.append("\nDRAM traffic per launch (read+write, bytes): " + ", ".join(f"{t:.4g}" for t in tr))
print("\n".join(out))
