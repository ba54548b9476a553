"""Per-source-line summary of an ncu --page source --csv (cuda,sass) export:
warp-stall samples and executed instructions, top N lines per file."""
import csv, gzip, sys, collections
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
op = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(op(path, "rt")))
cur_file = None
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, "", collections.Counter()])
hdr = None
tot_s = tot_i = 0.0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        hdr = None
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    try:
        s = float(r[4] or 0); ins = float(r[7] or 0); th = float(r[8] or 0)
    except ValueError:
        continue
    k = (cur_file, int(r[0]))
    a = agg[k]
    a[0] += s; a[1] += ins; a[2] += th; a[3] = r[1][:90]
    for i, n in enumerate(hdr):
        if n.startswith("stall_") and "Not Issued" not in n:
            try:
                a[4][n[6:]] += float(r[i] or 0)
            except ValueError:
                pass
    tot_s += s; tot_i += ins
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
byfile = collections.Counter()
for (f, l), a in agg.items():
    byfile[f] += a[0]
print("samples by file:", ", ".join(f"{f} {v/tot_s:.1%}" for f, v in byfile.most_common()))
for (f, l), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    st = ", ".join(f"{n} {v/a[0]:.0%}" for n, v in a[4].most_common(3)) if a[0] else ""
    eff = a[2] / a[1] if a[1] else 0
    print(f"{a[0]/tot_s:6.2%} {a[1]/tot_i:6.2%} eff {eff:4.1f} {f}:{l:<5d} {a[3]:90s} | {st}")
