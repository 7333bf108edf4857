timeout 300 python tools/panel_ab.py build_ab/lib_old.so paper_2503_17535_b200/libhps_b200.so > gpurun_out/panel_ab_512.jsonl 2>&1; echo "ab512 rc=$?"
timeout 300 python tools/panel_ab.py build_ab/lib_old.so build_ab/lib_r256.so > gpurun_out/panel_ab_256.jsonl 2>&1; echo "ab256 rc=$?"
cat gpurun_out/panel_ab_512.jsonl gpurun_out/panel_ab_256.jsonl
