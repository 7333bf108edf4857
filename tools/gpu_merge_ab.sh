timeout 300 python tools/fdm_check.py 8 > gpurun_out/merge_ab.jsonl 2>&1; echo "L8 rc=$?"; cut -c1-400 gpurun_out/merge_ab.jsonl
timeout 600 python tools/fdm_parity.py 8 > gpurun_out/merge_ab_par.jsonl 2>&1; echo "par rc=$?"; cat gpurun_out/merge_ab_par.jsonl | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_L8_m.csv python bench.py --profile --no-extras > gpurun_out/r02_ncu_launch_m.log 2>&1; echo "ncu rc=$?"
