bash tools/gpu_build_ab.sh build_ab/lib_noinv.so paper_2503_17535_b200/libhps_b200.so
timeout 600 python tools/fdm_parity.py 8 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
