# FP64 peak microbenchmark with SM clocks sampled during the run (profiles/r02_fp64_peak.json)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader,nounits -lms 50 > gpurun_out/fp64_clocks.csv 2>&1 &
SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak.out 2>&1
./tools/fp64_peak >> gpurun_out/fp64_peak.out 2>&1
kill $SMI
python - <<'PY'
import json
lines = [l for l in open('gpurun_out/fp64_peak.out') if l.startswith('{')]
res = {}
for l in lines:
    d = json.loads(l)
    for k, v in d.items():
        if isinstance(v, (int, float)): res.setdefault(k, []).append(v)
clk = [l.strip().split(',') for l in open('gpurun_out/fp64_clocks.csv') if l.strip() and l[0].isdigit()]
sm = sorted(float(c[0]) for c in clk)
out = {k: max(v) for k, v in res.items()}
out["clocks"] = {"sm_mhz_median": sm[len(sm) // 2] if sm else None, "sm_mhz_min": sm[0] if sm else None,
                 "sm_max_mhz": max(float(c[1]) for c in clk) if clk else None, "samples": len(sm),
                 "reasons": sorted({c[2].strip() for c in clk})}
out["note"] = "tools/fp64_peak.cu: DMMA (mma.sync m8n8k4 f64) and DFMA loops, best of 4 timed launches x 2 runs; the mixed figures issue both (they share the FP64 datapath)"
json.dump(out, open('gpurun_out/r02_fp64_peak.json', 'w'))
print(json.dumps(out))
PY
