"""Run the compression sweep (cmd_bench_cmax) on the GPU and print its rows.
usage: python tools/probes/cmax_sweep.py [H W dataset voxels]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2209_09965_b200.throughput import cmd_bench_cmax  # noqa: E402

h, w = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (180, 320)
ds = sys.argv[3] if len(sys.argv) > 3 else "vortex_field"
n = int(sys.argv[4]) if len(sys.argv) > 4 else 48
rows = cmd_bench_cmax(dims=(h, w), repeats=5, dataset=ds, volume_dims=(n, n, n), out_dir=ROOT / "gpurun_out")
print(f"{h}x{w} {ds} {n}^3: tau, t_naive_ms, t_compact_ms, c_max, t_full_ms, work_items")
for r in rows:
    print(f"  {r[0]:5.2f} {r[1]:8.3f} {r[2]:8.3f} {r[3]:6.3f} {r[4]:8.3f} {r[5]:8d}")
