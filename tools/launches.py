"""Summarise an ncu --metrics gpu__time_duration.sum launch list: the last frame's kernels."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
names = [(d["Kernel Name"], float(d["Metric Value"])) for d in data]
starts = [i for i, (n, _) in enumerate(names) if "mask_compact" in n]
last = names[starts[-1]:]
tot = sum(t for _, t in last)
agg = {}
for n, t in last:
    short = n.split("(")[0].replace("void ", "").replace("fv::<unnamed>::", "")
    print(f"{t / 1e3:9.1f} us  {short}")
    agg[short] = agg.get(short, 0) + t
print(f"total {tot / 1e6:.3f} ms over {len(last)} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {v / tot * 100:5.1f}%  {v / 1e3:9.1f} us  {k}")
