"""Hottest SASS instructions (warp-stall samples) of one kernel in an ncu report.

usage: python tools/ncu_sass_hot.py REPORT.ncu-rep KERNEL_REGEX [N]
Prints the N instructions with the most stall samples (share of the kernel's samples) and the
totals, from `ncu --page source --print-source sass`.
"""
import csv
import io
import subprocess
import sys


def load(rep, kern, what):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                          "--print-source", what], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] in ("Address", "Line No", "#"))
    return rows[hi], [r for r in rows[hi + 1:] if len(r) == len(rows[hi]) and r[0] != rows[hi][0]]


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    h, data = load(rep, kern, "sass")
    iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
    f = lambda v: float(v) if v not in ("", None) else 0.0
    tot, totE = sum(f(r[iS]) for r in data), sum(f(r[iE]) for r in data)
    print(f"stall samples {tot:.0f}  warp instructions {totE:.0f}  sass lines {len(data)}")
    for r in sorted(data, key=lambda r: -f(r[iS]))[:n]:
        print(f"{r[0]:>8} {f(r[iS]) / tot * 100:5.1f}% {f(r[iE]):>10.0f}  {r[iSrc][:70]}")


if __name__ == "__main__":
    main()
