set -u
python -m pytest tests/test_gpu_configs.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > gpurun_out/r26_tests.txt
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in cur k5e cur k5e; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C5 2>&1 | tail -1)" >> gpurun_out/r26_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r26_tests.txt gpurun_out/r26_ab.txt
