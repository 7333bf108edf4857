timeout 1200 python tools/adaptive_probe.py > gpurun_out/r02_adaptive.jsonl 2> gpurun_out/r02_adaptive.err; echo "rc=$?"
cat gpurun_out/r02_adaptive.jsonl; tail -5 gpurun_out/r02_adaptive.err
timeout 600 python -m pytest tests/test_gpu_general.py tests/test_gpu_ref_parity.py -m gpu -q -k "general or dump or iti" 2>&1 | tail -3
