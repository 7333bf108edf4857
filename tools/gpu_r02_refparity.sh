nproc > gpurun_out/r02_nproc.txt; free -g >> gpurun_out/r02_nproc.txt
timeout 900 python -m pytest tests/test_gpu_ref_parity.py tests/test_gpu_parity.py -m gpu -q -k "ref or L7 or config4 or solution_parity" --durations=15 > gpurun_out/r02_gpu_refparity.log 2>&1; echo "rc=$?"
tail -40 gpurun_out/r02_gpu_refparity.log
