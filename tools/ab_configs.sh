for c in C1 C3 C4 C5; do echo "new $(timeout 120 python tools/run_config.py --config $c --time 2>&1 | tail -1 | cut -c1-140)"; done
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/new.so; cp ab_old/libkohler_cuda.so paper_1707_05062_b200/lib/libkohler_cuda.so
for c in C1 C3 C4 C5; do echo "old $(timeout 120 python tools/run_config.py --config $c --time 2>&1 | tail -1 | cut -c1-140)"; done
cp /tmp/new.so paper_1707_05062_b200/lib/libkohler_cuda.so
