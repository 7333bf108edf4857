# round-2 verification run: GPU test suite, then the default bench (device + e2e + extras + CPU arms)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_gputests.log
timeout 1200 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r02_bench.err
