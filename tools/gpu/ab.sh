# A/B of library builds under abl/: tools/gpu/ab.sh "v1 v2 ..." [configs] [reps]
# Each variant: smoke parity check once, then ab_time interleaved `reps` times.
set -u
VARS="$1"; CFG="${2:-C2,C3,C4,C5}"; REPS="${3:-2}"
OUT=gpurun_out/ab_$(date +%H%M%S).txt
for v in $VARS; do
  KOHLER_CUDA_LIB=$PWD/abl/$v.so python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | sed "s/^/$v /" >> $OUT
done
for r in $(seq $REPS); do for v in $VARS; do
  echo "$v $(KOHLER_CUDA_LIB=$PWD/abl/$v.so python tools/ab_time.py --configs $CFG 2>&1 | tail -1)" >> $OUT
done; done
cat $OUT
