# select256_kernel occupancy A/B on C5 (K5 + K4 per batch)
set -u
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
cp paper_1707_05062_b200/lib/libkohler_cuda.so abl/cur.so
for v in cur sel4 sel5 sel6 cur sel4 sel5 sel6; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C5 2>&1 | tail -1)" >> gpurun_out/r23_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r23_ab.txt
