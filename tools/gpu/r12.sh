# self-finishing K1 (single images): full GPU suite, A/B base vs sf1 on C1/C2/C4, bench line
set -u
python -m pytest tests -q -m gpu -x 2>&1 | tail -8 > gpurun_out/r12_gpu_suite.txt
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in base sf1 base sf1; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C1,C2,C4 2>&1 | tail -1)" >> gpurun_out/r12_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
python bench.py --steps 20 --warmup 5 > gpurun_out/r12_bench.json 2> gpurun_out/r12_bench.err
cat gpurun_out/r12_gpu_suite.txt gpurun_out/r12_ab.txt; cut -c1-400 gpurun_out/r12_bench.json
