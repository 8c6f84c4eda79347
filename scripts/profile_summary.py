"""Summarise an ncu --set full report (per-kernel metrics) and a launch-list CSV into
profiles/ (markdown + json).  Usage: profile_summary.py <rep | raw.csv> <launches.csv> <out_prefix>
<label> [hot_lines.txt]   (a *_raw.csv is the `ncu -i rep --page raw --csv` export that
scripts/gpu_round.sh writes on the box; the optional hot-lines text is appended)"""
import csv, io, json, os, subprocess, sys
rep, launches, out, label = sys.argv[1:5]
hot = sys.argv[5] if len(sys.argv) > 5 else None
if rep.endswith(".csv"):
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__inst_executed_pipe_fp64.sum",
        "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
want += [h for h in rows[0] if h.startswith("smsp__average_warps_issue_stalled_") and
         h.endswith("_per_issue_active.ratio")]
idx = {k: hdr.index(k) for k in want if k in hdr}
kern = []
for r in data:
    kern.append({k: (r[i] if i < len(r) else None) for k, i in idx.items()})
summ = {"label": label, "kernels": kern, "units": {k: units[i] for k, i in idx.items()}}
# launch list
L = []
try:
    rows = [r for r in csv.reader(open(launches)) if r]
    h = None
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            h = r; continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                L.append((d["Kernel Name"], float(d["Metric Value"].replace(",", ""))))
except FileNotFoundError:
    pass
agg = {}
for k, v in L:
    name = k.split("(")[0]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1; a[1] += v
tot = sum(v for _, v in agg.values()) or 1.0
summ["launch_list"] = {k: {"launches": n, "total_ns": t, "share": t / tot} for k, (n, t) in agg.items()}
json.dump(summ, open(out + ".json", "w"), indent=1)
with open(out + ".md", "w") as f:
    f.write("# ncu summary: %s\n\n" % label)
    f.write("## launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n\n")
    f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
    for k, d in sorted(summ["launch_list"].items(), key=lambda x: -x[1]["total_ns"]):
        f.write("| %s | %d | %.3f | %.1f%% |\n" % (k, d["launches"], d["total_ns"] / 1e6, 100 * d["share"]))
    f.write("\n## --set full capture\n\n")
    for k in kern:
        f.write("### %s\n\n" % k.get("Kernel Name"))
        for m, v in k.items():
            if m != "Kernel Name":
                f.write("- %s = %s %s\n" % (m, v, summ["units"].get(m, "")))
        f.write("\n")
    if hot and os.path.exists(hot):
        f.write("## hottest source lines (warp-stall samples; scripts/ncu_hot_lines.py)\n\n```\n")
        f.write("".join(open(hot).readlines()[:41]))
        f.write("```\n")
print(open(out + ".md").read())
