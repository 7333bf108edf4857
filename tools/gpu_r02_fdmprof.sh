# FDM leaf default: GPU bench (default run), launch list of one profiled step, ncu --set full of leaf_fdm_kernel
timeout 1500 python bench.py > gpurun_out/r02_bench3.json 2> gpurun_out/r02_bench3.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r02_bench3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_L8_fdm.csv python bench.py --profile --no-extras --no-cpu-baseline > gpurun_out/r02_ncu_launch_fdm.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaf_fdm_kernel -c 1 -o gpurun_out/r02_fdm_full python tools/leaf_prof.py > gpurun_out/r02_fdm_full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/r02_fdm_full.log
