"""Per-source-line warp-stall roll-up of an ncu --set full report (developer tool).
usage: python tools/ncu_hot.py report.ncu-rep [top]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur = None; hdr = None; out = []
for r in rows:
    if r and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr and r and r[0] not in ('', 'Function Name'):
        try: s = int(r[4])
        except (ValueError, IndexError): continue
        g = lambda k: r[hdr.index(k)] if k in hdr else '?'
        out.append((s, cur, r[0], r[1].strip()[:80], g('stall_wait'), g('stall_short_sb'), g('stall_barrier'),
                    g('stall_long_sb'), g('stall_math')))
tot = sum(o[0] for o in out) or 1
print('total samples', tot)
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0]:8d} {100*o[0]/tot:5.1f}% {o[1]}:{o[2]} wait={o[4]} ssb={o[5]} bar={o[6]} lsb={o[7]} math={o[8]} | {o[3]}")
