timeout 900 python -m pytest tests -m gpu -q -k "iti or radiation or general or scatter" > gpurun_out/r02_iti.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/r02_iti.log
python - <<'PY' > gpurun_out/r02_iti_bench.txt 2>&1
import sys, time; sys.path.insert(0, '.')
import bench, argparse, torch
print(bench.bench_iti(torch))
PY
cat gpurun_out/r02_iti_bench.txt
