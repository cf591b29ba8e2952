# cluster-reduced small single images: new tests, full suite, A/B on C1/C2
set -u
python -m pytest tests/test_gpu_single_paths.py -q -x 2>&1 | tail -15 > gpurun_out/r14_single.txt
python -m pytest tests -q -m gpu -x 2>&1 | tail -8 > gpurun_out/r14_gpu_suite.txt
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in base cl2 base cl1; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C1,C2 2>&1 | tail -1)" >> gpurun_out/r14_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
echo "cl2 no-cluster $(KOHLER_NO_CLUSTER=1 python tools/ab_time.py --configs C1 2>&1 | tail -1)" >> gpurun_out/r14_ab.txt
cat gpurun_out/r14_single.txt gpurun_out/r14_gpu_suite.txt gpurun_out/r14_ab.txt
