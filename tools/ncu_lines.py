"""Per-CUDA-line instruction and stall-sample shares of one kernel in an ncu report.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N] [--by inst|stall]
From `ncu --page source --print-source cuda,sass`: each source line's share of the kernel's
executed warp instructions and warp-stall samples, and its two largest stall reasons.
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
    by = "stall" if "stall" in sys.argv[3:] else "inst"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    reasons = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    f = lambda v: float(v) if v not in ("", "-", None) else 0.0
    lines = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] not in ("", "Line No")]
    tot, totE = sum(f(r[iS]) for r in lines), sum(f(r[iE]) for r in lines)
    print(f"stall samples {tot:.0f}  warp instructions {totE:.0f}")
    key = (lambda r: -f(r[iE])) if by == "inst" else (lambda r: -f(r[iS]))
    for r in sorted(lines, key=key)[:n]:
        rs = sorted(((f(r[i]), c[6:]) for i, c in reasons), reverse=True)[:2]
        why = " ".join(f"{c}:{v / max(f(r[iS]), 1) * 100:.0f}%" for v, c in rs if v)
        print(f"{r[0]:>5} inst {f(r[iE]) / totE * 100:5.1f}%  stall {f(r[iS]) / tot * 100:5.1f}%  {why:28s} {r[1].strip()[:70]}")


if __name__ == "__main__":
    main()
