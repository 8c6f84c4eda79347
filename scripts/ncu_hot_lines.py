"""Top source lines of an ncu report by warp-stall samples (cuda source view).
Usage: ncu_hot_lines.py <rep> [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] in ("File Path", "File Name"): fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0] != "":
        d = dict(zip(hdr[2:], r[2:])); d["Line No"] = r[0]; d["Source"] = r[1]
        try: s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError: continue
        try: ins = int(d.get("Instructions Executed", "0") or 0)
        except ValueError: ins = 0
        rows.append((s, ins, fname, d["Line No"], d["Source"].strip()[:110]))
tot = sum(x[0] for x in rows) or 1
print("total samples", tot)
for s, ins, f, ln, src in sorted(rows, reverse=True)[:N]:
    print("%5.1f%% %12d %s:%s  %s" % (100 * s / tot, ins, f, ln, src))
