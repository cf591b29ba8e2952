# round-2 GPU call: new parity tests + compute-sanitizer runs (small shapes)
mkdir -p gpurun_out/san
python -m pytest tests/test_gpu_adversarial.py tests/test_gpu_nccl_bands.py -x -q 2>&1 | tail -15 > gpurun_out/r2_tests.txt
python -m pytest tests/test_gpu_configs.py -x -q -k c3 2>&1 | tail -5 >> gpurun_out/r2_tests.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 99 python tools/sanitize_small.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/summary.txt
done
cat gpurun_out/r2_tests.txt gpurun_out/san/summary.txt
