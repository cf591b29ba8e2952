set -u
python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/r30_tests.txt
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in cur fuse1 cur fuse1; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C5 2>&1 | tail -1)" >> gpurun_out/r30_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r30_tests.txt gpurun_out/r30_ab.txt
