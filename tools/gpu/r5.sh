python -m pytest tests -q -m gpu -x 2>&1 | tail -8 > gpurun_out/r5_gpu_suite.txt
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in base nosync base nosync; do cp ab/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C2,C4,C5 2>&1 | tail -1)" >> gpurun_out/r5_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r5_gpu_suite.txt gpurun_out/r5_ab.txt
