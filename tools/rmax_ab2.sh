# A/B of -DKOHLER_MAX_WALK_ROWS builds (ab_old/r192.so, ab_old/r256.so, built here with nvcc) against the
# working-tree library (128): C2 bench line and C4 device timing, same box.
cd $GRAFT_REPO_ROOT
L=paper_1707_05062_b200/lib/libkohler_cuda.so
cp $L /tmp/r128.so
for v in r128 r192 r256 r128; do
  if [ $v = r128 ]; then cp /tmp/r128.so $L; else cp ab_old/$v.so $L; fi
  b=$(timeout 300 python bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")
  c4=$(timeout 120 python tools/run_config.py --config C4 --time 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['gpix_per_s'],1))")
  echo "$v bench $b C4 $c4"
done
cp /tmp/r128.so $L
