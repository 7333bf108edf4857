# one panel launch (n=1792 batch 16, second case index) of each variant under ncu --set full
cat > /tmp/one.py <<'PY'
import sys, ctypes as C, torch
L = C.CDLL(sys.argv[1])
L.hpsg_dev_getrf_aug.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p, C.c_void_p]
n, m, b = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
g = torch.Generator(device="cuda").manual_seed(n)
M = torch.randn((b, n + m, n), dtype=torch.float64, device="cuda", generator=g)
piv = torch.zeros((b, n), dtype=torch.int32, device="cuda"); st = torch.zeros((b, 3), dtype=torch.float64, device="cuda")
print(L.hpsg_dev_getrf_aug(b, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), st.data_ptr()))
PY
timeout 300 ncu --set full --clock-control none --import-source on -k regex:panel_getrf -s 2 -c 1 -o gpurun_out/panel_old python /tmp/one.py build_ab/lib_old.so 1792 3585 16 > gpurun_out/panel_old.log 2>&1; echo "old rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:panel_getrf -s 2 -c 1 -o gpurun_out/panel_new python /tmp/one.py paper_2503_17535_b200/libhps_b200.so 1792 3585 16 > gpurun_out/panel_new.log 2>&1; echo "new rc=$?"
