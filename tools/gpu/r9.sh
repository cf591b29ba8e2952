# K5 phases (per-CTA cycles) base vs new on uniform and C5-family data; ncu of the new K5
set -u
for f in 0 1; do
  echo "fam $f base: $(abl/tile_probe_base 65536 128 128 $f | tail -2 | tr '\n' ' ')" >> gpurun_out/r9_phases.txt
  echo "fam $f new : $(tools/tile_probe 65536 128 128 $f | tail -2 | tr '\n' ' ')" >> gpurun_out/r9_phases.txt
done
timeout 500 ncu --set full --import-source on --clock-control none -k regex:twalk_kernel -s 1 -c 1 -o gpurun_out/r9_c5_twalk python tools/run_config.py --config C5 --reps 2 > gpurun_out/r9_ncu_c5.log 2>&1
cat gpurun_out/r9_phases.txt
