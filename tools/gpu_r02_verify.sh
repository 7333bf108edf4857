# full verification: GPU suite, default bench, launch list of one profiled step
TAG=${1:-v6}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests_${TAG:-v6}.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02_gputests_${TAG:-v6}.log
timeout 1800 python bench.py > gpurun_out/r02_bench_${TAG:-v6}.json 2> gpurun_out/r02_bench_${TAG:-v6}.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r02_bench_${TAG:-v6}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_L8_${TAG:-v6}.csv python bench.py --profile --no-extras > gpurun_out/r02_ncu_launch_${TAG:-v6}.log 2>&1; echo "ncu rc=$?"
