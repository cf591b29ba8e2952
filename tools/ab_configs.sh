# A/B timing of the working-tree library against ab_old/libkohler_cuda.so
# (built from the previous commit); same box, interleaved.
set -u
run() { for c in C2 C3 C4 C5; do d=1; [ $c = C2 ] && d=2; echo "$1 $(timeout 120 python tools/run_config.py --config $c --time --depth $d 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d[\"config\"], round(d[\"gpix_per_s\"],1))")"; done; }
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/new.so
for rep in 1 2; do
  cp /tmp/new.so paper_1707_05062_b200/lib/libkohler_cuda.so; run new
  cp ab_old/libkohler_cuda.so paper_1707_05062_b200/lib/libkohler_cuda.so; run old
done
cp /tmp/new.so paper_1707_05062_b200/lib/libkohler_cuda.so
