set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_box.txt 2>&1
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputests.log 2>&1; echo "pytest rc=$?"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck racecheck; do
  for part in leaf lu gemm; do
    timeout 600 $CS --tool $tool --print-limit 20 python tools/sanitize.py $part > gpurun_out/r02_sanitizer_${tool}_${part}.txt 2>&1
    echo "$tool $part rc=$?"
  done
done
