# FDM leaf kernel iteration: parity + timing + ncu of the new kernel + FP64 pipe co-issue probe
rm -f gpurun_out/fdm_check2.jsonl gpurun_out/fdm_parity2.jsonl
./tools/fp64_peak > gpurun_out/fp64_mixed.json 2>&1; cat gpurun_out/fp64_mixed.json
for L in 3 5 8; do timeout 300 python tools/fdm_check.py $L >> gpurun_out/fdm_check2.jsonl 2>> gpurun_out/fdm_check2.err; echo "fdm L=$L rc=$?"; done
timeout 600 python tools/fdm_parity.py 8 >> gpurun_out/fdm_parity2.jsonl 2>> gpurun_out/fdm_parity2.err; echo "parity rc=$?"
cat gpurun_out/fdm_check2.jsonl gpurun_out/fdm_parity2.jsonl | cut -c1-400; tail -c 600 gpurun_out/fdm_check2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:leaf_fdm_kernel -c 1 -o gpurun_out/r02_fdm_full2 python tools/leaf_prof.py > gpurun_out/r02_fdm_full2.log 2>&1; echo "ncu rc=$?"
