"""Per-launch table of an `ncu --set full` report: duration, DRAM bytes, tensor/L1/L2 utilisation.

usage: python tools/ncu_table.py REPORT.ncu-rep [--json OUT.json --key NAME]
Prints a markdown table (one row per captured launch) and, with --json, merges
{"NAME": {"dram_bytes_per_launch": mean, "launches": n, ...}} into OUT.json (the
`roofline.traffic` source read by bench.py).
"""
import argparse
import csv
import json
import subprocess
from pathlib import Path

METRICS = {
    "us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "tensor%": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "smem_tc%": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1%": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l2%": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "issue%": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
         "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}


def rows(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units, data = r[0], r[1], r[2:]
    col = {k: (hdr.index(m) if m in hdr else None) for k, m in METRICS.items()}
    ki = hdr.index("Kernel Name")
    res = []
    for d in data:
        e = {"kernel": d[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")}
        for k, i in col.items():
            if i is None or not d[i]:
                e[k] = None
                continue
            try:
                v = float(d[i].replace(",", ""))
            except ValueError:  # "no data" / "n/a"
                e[k] = None
                continue
            if k.startswith("dram_") or k == "us":
                v *= SCALE.get(units[i], 1.0)
            e[k] = v
        res.append(e)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--json")
    ap.add_argument("--key")
    a = ap.parse_args()
    rs = rows(a.report)
    cols = list(METRICS)
    print("| # | kernel | " + " | ".join(cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    for i, e in enumerate(rs):
        cells = []
        for c in cols:
            v = e[c]
            if v is None:
                cells.append("-")
            elif c.startswith("dram_"):
                cells.append(f"{v / 1e6:.1f} MB")
            else:
                cells.append(f"{v:.1f}")
        print(f"| {i} | {e['kernel']} | " + " | ".join(cells) + " |")
    tot_us = sum(e["us"] for e in rs)
    tot_b = sum((e["dram_rd"] or 0) + (e["dram_wr"] or 0) for e in rs)
    print(f"\n{len(rs)} launches, {tot_us:.1f} us, DRAM {tot_b / 1e6:.1f} MB "
          f"({tot_b / len(rs) / 1e6:.1f} MB per launch)")
    if a.json:
        p = Path(a.json)
        j = json.loads(p.read_text()) if p.exists() else {}
        j[a.key] = {"dram_bytes_per_launch": tot_b / len(rs), "launches": len(rs), "sum_us": tot_us,
                    "report": Path(a.report).name,
                    "note": "dram__bytes_read.sum + dram__bytes_write.sum averaged over the captured launches "
                            "(ncu --set full, cache control all = cold L2 per launch)"}
        p.write_text(json.dumps(j, indent=1) + "\n")


if __name__ == "__main__":
    main()
