"""Summarise gpurun_out/timeline.json: per-frame net/march kernel time, net gaps, and one frame's kernels."""
import json, re, sys
ev = json.load(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/timeline.json'))
ev = [e for e in ev if e['cat'] == 'kernel']
ev.sort(key=lambda e: e['ts'])
net_s = max(set(e['stream'] for e in ev), key=lambda s: sum(1 for e in ev if e['stream'] == s))
allev = json.load(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/timeline.json'))
bounds = sorted(e['ts'] for e in allev if e['cat'] == 'gpu_memcpy' and 'HtoD' in e['name'])
def short(n):
    n = re.sub(r'void |fv::|\(anonymous namespace\)::|<unnamed>::', '', n)
    return n[:60]
rows = []
for a, b in zip(bounds, bounds[1:]):
    fr = [e for e in ev if a <= e['ts'] < b]
    net = sum(e['dur'] for e in fr if e['stream'] == net_s)
    oth = sum(e['dur'] for e in fr if e['stream'] != net_s)
    nv = sorted((e['ts'], e['ts'] + e['dur']) for e in fr if e['stream'] == net_s)
    gaps = sum(max(0, nv[i + 1][0] - nv[i][1]) for i in range(len(nv) - 1))
    rows.append((b - a, net, oth, gaps))
    print(f"frame {b-a:7.1f} us: net kernels {net:7.1f}, march-branch kernels {oth:6.1f}, net gaps {gaps:6.1f}")
if len(bounds) > 3:
    a, b = bounds[len(bounds) // 2], bounds[len(bounds) // 2 + 1]
    for e in ev:
        if a <= e['ts'] < b:
            print(f"{e['ts']-a:9.1f} {e['dur']:7.1f} {'N' if e['stream']==net_s else 'M'} {short(e['name'])}")
