python tools/leaf_ab.py build_ab/libhps_b200_gepp0.so 8
python tools/leaf_ab.py paper_2503_17535_b200/libhps_b200.so 8
python tools/leaf_ab.py build_ab/libhps_b200_gepp0.so 8
python tools/leaf_ab.py paper_2503_17535_b200/libhps_b200.so 8
python -c "
import numpy as np
a=np.load('gpurun_out/leaf_ab_u_libhps_b200_gepp0.so_8.npy'); b=np.load('gpurun_out/leaf_ab_u_libhps_b200.so_8.npy')
print('u diff new vs old', np.abs(a-b).max()/np.abs(a).max())"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_parity.py -m gpu -q -x -k "fused or artifact or solution_parity or dtn_vs or node_artifacts" 2>&1 | tail -3
