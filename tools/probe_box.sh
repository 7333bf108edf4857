#!/bin/bash
# One-shot GPU-box probe: host cores/RAM, FP64 peaks (DMMA/DFMA microbench, cuBLAS DGEMM).
set -x
mkdir -p gpurun_out
nproc; lscpu | head -20; free -g; nvidia-smi
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak | tee gpurun_out/fp64_peak.json
python - <<'PY' | tee gpurun_out/dgemm.json
import torch, json
n=8192
a=torch.randn(n,n,dtype=torch.float64,device='cuda'); b=torch.randn(n,n,dtype=torch.float64,device='cuda')
for _ in range(3): c=a@b
torch.cuda.synchronize()
best=1e9
for _ in range(5):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); c=a@b; e.record(); torch.cuda.synchronize(); best=min(best,s.elapsed_time(e))
print(json.dumps({"cublas_dgemm_8192_tflops": 2*n**3/best/1e9, "ms": best}))
PY
