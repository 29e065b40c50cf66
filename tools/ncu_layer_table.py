"""Markdown tables from the raw-page CSVs of the round-2 ncu captures (tools/probes/evidence_r02b.sh):
one row per captured launch with duration, DRAM bytes, tensor-pipe / smem-operand / DRAM utilisation
and the SM-active fraction (cycles with a resident warp / elapsed cycles).

usage: python tools/ncu_layer_table.py RAW.csv [layer names ...] > table.md"""
import csv
import sys

COLS = [
    ("us", "gpu__time_duration.sum", 1.0),
    ("DRAM rd MB", "dram__bytes_read.sum", 1.0),
    ("DRAM wr MB", "dram__bytes_write.sum", 1.0),
    ("tensor pipe %", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("smem->TC %", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
    ("L1/TEX %", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0),
    ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("issue %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    ("tcgen05.mma", "sm__inst_executed_pipe_tensor_subpipe_hmma.sum", 1.0),
]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {k: i for i, k in enumerate(hdr)}
    names = sys.argv[2:]
    head = ["#", "layer", "kernel"] + [c[0] for c in COLS] + ["SM active %"]
    print("| " + " | ".join(head) + " |")
    print("|" + "---|" * len(head))
    for n, r in enumerate(data):
        k = r[idx["Kernel Name"]].replace("void ", "").replace("fv::", "").replace("(anonymous namespace)::", "")
        k = k.replace("<unnamed>::", "").replace("unnamed>::", "").split("(")[0]
        vals = []
        for _, m, _s in COLS:
            v = r[idx[m]] if m in idx else ""
            try:
                f = float(v.replace(",", ""))
                vals.append(f"{f:.0f}" if f >= 1000 else f"{f:.1f}")
            except ValueError:
                vals.append("-")
        act = "-"
        if "smsp__cycles_active.avg" in idx and "sm__cycles_elapsed.avg" in idx:
            try:
                act = f"{100 * float(r[idx['smsp__cycles_active.avg']]) / float(r[idx['sm__cycles_elapsed.avg']]):.0f}"
            except ValueError:
                pass
        layer = names[n] if n < len(names) else ""
        print(f"| {n} | {layer} | `{k}` | " + " | ".join(vals) + f" | {act} |")


if __name__ == "__main__":
    main()
