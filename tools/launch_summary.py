"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel and by build phase."""
import csv, collections, sys
path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0.0; seq = []
for r in rows[1:]:
    if r[0] == "ID": continue
    v = float(r[idx['Metric Value']].replace(',', ''))
    name = r[idx['Kernel Name']].replace('(anonymous namespace)::', '').replace('hpsk::', '')
    short = name.split('(')[0]
    for pre in ('void ', 'unnamed>::'): short = short.replace(pre, '')
    agg[short][0] += 1; agg[short][1] += v; tot += v
    seq.append((short, v, r[idx['Grid Size']], r[idx['Block Size']]))
print(f"{'kernel':55s} {'launches':>8s} {'ms':>10s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:55]:55s} {n:8d} {t/1e6:10.2f} {100*t/tot:5.1f}%")
print(f"total {tot/1e6:.2f} ms over {len(seq)} launches")
if len(sys.argv) > 2:
    # top individual launches
    for s in sorted(seq, key=lambda x: -x[1])[:int(sys.argv[2])]:
        print(f"  {s[0][:50]:50s} {s[1]/1e6:8.3f} ms grid {s[2]} block {s[3]}")

# per-phase breakdown: grid.x is the batch (nodes of the level; x cluster size for panels)
phase = collections.defaultdict(lambda: collections.defaultdict(float))
cur = "leaf"
for name, v, grid, blk in seq:
    g = grid.strip("()").split(",")
    gx = int(g[0])
    if name.startswith("gather"):
        cur = f"merge batch={gx}"
    phase[cur][name.split("<")[0]] += v
print("\nper phase (ms):")
for ph, d in phase.items():
    print(f"  {ph:22s} total {sum(d.values())/1e6:8.2f}  " + "  ".join(f"{k}={t/1e6:.2f}" for k, t in sorted(d.items(), key=lambda x: -x[1])))
