set -u
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in cur g47 g46 cur g47 g46; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C2 2>&1 | tail -1) $(python bench.py --steps 20 --warmup 5 --no-per-config 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))')" >> gpurun_out/r21_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r21_ab.txt
