for L in 6 7 8; do timeout 600 python tools/fdm_parity.py $L >> gpurun_out/fdm_parity.jsonl 2>> gpurun_out/fdm_parity.err; echo "L=$L rc=$?"; done
cat gpurun_out/fdm_parity.jsonl; tail -c 600 gpurun_out/fdm_parity.err
