"""Per-kernel counts of the SASS mnemonics that prove the bulk-copy / TMA, mbarrier and
tcgen05 paths (B200_PROFILING.md): UBLKCP (cp.async.bulk), UTMALDG (TMA tensor load),
SYNCS (mbarrier ops), UTC*MMA (tcgen05.mma), LDTM (tcgen05.ld), plus a few sample lines.
Usage: sass_summary.py <cuobjdump -sass output>"""
import collections, re, sys

MN = ("UBLKCP", "UTMALDG", "UTMAPF", "SYNCS", "UTCHMMA", "UTCQMMA", "UTCMMA", "UTCBAR", "LDTM",
      "STTM", "DFMA", "MUFU")
fn, counts, samples = None, collections.OrderedDict(), collections.defaultdict(list)
for line in open(sys.argv[1], errors="replace"):
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        counts[fn] = collections.Counter()
        continue
    if fn is None or "/*" not in line:
        continue
    ins = line.split("*/", 1)[-1].strip()
    for k in MN:
        if re.search(r"\b" + k + r"[\.\s]", ins + " "):
            counts[fn][k] += 1
            if len(samples[(fn, k)]) < 2:
                samples[(fn, k)].append(ins[:120])
for fn, c in counts.items():
    if not c:
        continue
    print(fn)
    print("   " + "  ".join("%s=%d" % kv for kv in sorted(c.items())))
    for k in MN:
        for s in samples.get((fn, k), []):
            print("      " + s)
