# FDM leaf path check: artifacts/solution vs the LU leaf path, leaf-stage times; then the GPU suite
for L in 3 5 8; do timeout 300 python tools/fdm_check.py $L >> gpurun_out/fdm_check.jsonl 2>> gpurun_out/fdm_check.err; echo "fdm L=$L rc=$?"; done
tail -c 1500 gpurun_out/fdm_check.jsonl; tail -c 800 gpurun_out/fdm_check.err
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02_gputests_fdm.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02_gputests_fdm.log
