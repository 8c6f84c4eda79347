"""Aggregate an ncu source page (cuda,sass csv) into per-source-line stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur = None; hdr = None; lines = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if len(r) >= 2 and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 6: continue
    if r[0] != "":
        try: lines.append((cur, int(r[0]), r[1].strip(), float(r[4] or 0), float(r[5] or 0)))
        except Exception: pass
tot = sum(l[3] for l in lines)
print("total samples", tot)
for l in sorted(lines, key=lambda x: -x[3])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print("%5.1f%% %5.1f%% %-10s %5d %s" % (100*l[3]/tot, 100*l[4]/tot, l[0][:10], l[1], l[2][:100]))
