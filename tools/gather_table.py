"""Summarise tools/gather_prof.sh output: per-launch time, DRAM bytes, bandwidth (developer tool)."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
I = {k: i for i, k in enumerate(rows[0])}
d = defaultdict(dict)
for r in rows[1:]:
    d[r[I['ID']]][r[I['Metric Name']]] = float(r[I['Metric Value']].replace(',', ''))
tt = 0
for k, v in sorted(d.items(), key=lambda x: int(x[0])):
    t = v['gpu__time_duration.sum']; rb = v['dram__bytes_read.sum']; wb = v['dram__bytes_write.sum']
    tt += t
    print(f"{k:>3} t_us={t/1e3:8.1f} rd={rb/1e6:7.1f}MB wr={wb/1e6:7.1f}MB GB/s={(rb+wb)/t:6.0f} "
          f"sm%={v['sm__throughput.avg.pct_of_peak_sustained_elapsed']:.0f}")
print(f"total {tt/1e6:.2f} ms")
