"""Top CUDA-C source lines by stall samples from `ncu -i rep --page source --print-source cuda,sass --csv` (gz).
usage: python tools/ncu_srclines.py file.csv.gz [top N] [launch index]"""
import collections, csv, gzip, io, sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(io.TextIOWrapper(gzip.open(path), newline="")))
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
cur_file, hdr, ix = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        hdr = None
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {}
        for i, h in enumerate(r):
            ix.setdefault(h, i)
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].strip().isdigit() or r[2] != "-":
        continue
    samp, ex = int(r[ix["# Samples"]]), int(r[ix["Instructions Executed"]])
    key = (cur_file, int(r[0]), r[1].strip()[:100])
    agg[key][0] += samp
    agg[key][1] += ex
    for h, i in ix.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            v = int(r[i] or 0)
            if v:
                agg[key][2][h[6:]] += v
tot = sum(v[0] for v in agg.values())
print("total samples (all captured launches)", tot, "source lines", len(agg))
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{k[0]}:{k[1]:5d} samp {v[0]:5d} ({100.0 * v[0] / max(tot, 1):4.1f}%) exec {v[1]:8d} {dict(v[2].most_common(3))} | {k[2]}")
