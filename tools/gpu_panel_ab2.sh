timeout 300 python tools/panel_ab.py build_ab/lib_old.so paper_2503_17535_b200/libhps_b200.so > gpurun_out/panel_ab_nbt.jsonl 2>&1; echo "ab rc=$?"
cat gpurun_out/panel_ab_nbt.jsonl
timeout 300 python tools/fdm_check.py 8 > gpurun_out/fdm_check_nbt.jsonl 2>&1; echo "L8 rc=$?"; cut -c1-250 gpurun_out/fdm_check_nbt.jsonl
