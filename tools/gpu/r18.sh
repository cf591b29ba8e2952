# K1 occupancy probe: 512 (4 warps/SMSP), 384 (3), 256 (2) threads per CTA
set -u
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in cur t384 t256 cur t384 t256; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C2,C3,C4 2>&1 | tail -1)" >> gpurun_out/r18_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r18_ab.txt
