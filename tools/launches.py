"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: python tools/launches.py LAUNCHES.csv [--markdown]
Frames start at each mask_compact_kernel launch; the last (possibly truncated by ncu -c)
frame is dropped when more than one frame was captured. Prints the last complete frame's
launches and the per-kernel mean time per frame over all complete frames.
"""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    out = []
    for d in data:
        if d.get("Metric Name", "gpu__time_duration.sum") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "nsecond")
        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("fv::<unnamed>::", "")
        out.append((name.replace("<unnamed>::", "").replace("unnamed>::", ""), v))
    return out


def frames(launches):
    starts = [i for i, (n, _) in enumerate(launches) if n.startswith("mask_compact")]
    fr = [launches[a:b] for a, b in zip(starts, starts[1:] + [len(launches)])]
    return fr[:-1] if len(fr) > 1 else fr


def main():
    path = sys.argv[1]
    md = "--markdown" in sys.argv
    fr = frames(load(path))
    last = fr[-1]
    tot = sum(t for _, t in last)
    if md:
        print(f"Last complete frame ({len(last)} launches, {tot / 1e3:.3f} ms summed, serialised by ncu):\n")
        print("| # | kernel | us |\n|---|---|---|")
        for i, (n, t) in enumerate(last):
            print(f"| {i} | `{n}` | {t:.1f} |")
    else:
        for n, t in last:
            print(f"{t:9.1f} us  {n}")
        print(f"total {tot / 1e3:.3f} ms over {len(last)} launches")
    agg = {}
    for f in fr:
        for n, t in f:
            agg[n] = agg.get(n, 0.0) + t / len(fr)
    tt = sum(agg.values())
    if md:
        print(f"\nMean per frame over {len(fr)} complete frames ({tt / 1e3:.3f} ms):\n")
        print("| kernel | us/frame | share |\n|---|---|---|")
        for n, v in sorted(agg.items(), key=lambda x: -x[1]):
            print(f"| `{n}` | {v:.1f} | {v / tt * 100:.1f}% |")
    else:
        print(f"mean over {len(fr)} complete frames: {tt / 1e3:.3f} ms")
        for n, v in sorted(agg.items(), key=lambda x: -x[1]):
            print(f"  {v / tt * 100:5.1f}%  {v:9.1f} us  {n}")


if __name__ == "__main__":
    main()
