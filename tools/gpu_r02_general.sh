timeout 900 python -m pytest tests/test_gpu_general.py -m gpu -q -x > gpurun_out/r02_general.log 2>&1; echo "general rc=$?"; tail -30 gpurun_out/r02_general.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests2.log 2>&1; echo "all rc=$?"; tail -5 gpurun_out/r02_gputests2.log
