"""Headline counters of an ncu --set full report (developer tool): python tools/ncu_metrics.py report.ncu-rep"""
import csv, subprocess, sys, io
txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    print(d.get('Kernel Name', '')[:80])
    for k in ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
              'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active',
              'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
              'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
              'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem', 'launch__grid_size',
              'dram__throughput.avg.pct_of_peak_sustained_elapsed']:
        print(f"  {k} = {d.get(k, '?')}")
