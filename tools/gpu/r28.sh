set -u
python -m pytest tests/test_gpu_single_paths.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2 > gpurun_out/r28_tests.txt
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in cur fin2 cur fin2; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C1,C2 2>&1 | tail -1)" >> gpurun_out/r28_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r28_tests.txt gpurun_out/r28_ab.txt
