# ncu --set full of the first slab_trsm (depth 6, batch 4096, n = 112), the first gather and the depth-7 trsm_upper
timeout 600 ncu --set full --clock-control none --import-source on -k regex:slab_trsm -c 1 -o gpurun_out/r02_slab_trsm python tools/leaf_prof.py > gpurun_out/r02_slab.log 2>&1; echo "slab rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -c 1 -o gpurun_out/r02_gather python tools/leaf_prof.py > gpurun_out/r02_gather.log 2>&1; echo "gather rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsm_upper -c 1 -o gpurun_out/r02_trsmu python tools/leaf_prof.py > gpurun_out/r02_trsmu.log 2>&1; echo "trsmu rc=$?"
