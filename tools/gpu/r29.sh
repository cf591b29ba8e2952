set -u
python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > gpurun_out/r29_tests.txt
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in cur tw4 tw3 cur tw4 tw3; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C5 2>&1 | tail -1)" >> gpurun_out/r29_ab.txt; done
cp abl/tw3.so paper_1707_05062_b200/lib/libkohler_cuda.so
python -m pytest tests/test_gpu_configs.py -q -x -k c5 2>&1 | tail -2 >> gpurun_out/r29_tests.txt
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r29_tests.txt gpurun_out/r29_ab.txt
