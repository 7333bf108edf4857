timeout 300 python tools/solve_ab.py build_ab/lib_trsv1.so /tmp/u_old.npy; timeout 300 python tools/solve_ab.py paper_2503_17535_b200/libhps_b200.so /tmp/u_new.npy
python -c "import numpy as np; a=np.load('/tmp/u_old.npy'); b=np.load('/tmp/u_new.npy'); print('bitwise', np.array_equal(a,b), 'maxdiff', float(np.abs(a-b).max()))"
