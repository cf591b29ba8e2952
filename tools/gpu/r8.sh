# K5 flush rework: GPU suite on the new library, then A/B timing base vs new (interleaved)
set -u
python -m pytest tests -q -m gpu -x 2>&1 | tail -6 > gpurun_out/r8_gpu_suite.txt
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in base k5a base k5a; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C5,C2 2>&1 | tail -1)" >> gpurun_out/r8_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r8_gpu_suite.txt gpurun_out/r8_ab.txt
