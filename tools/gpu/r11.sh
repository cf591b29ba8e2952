set -u
python -m pytest tests -q -m gpu -x -k "c5 or C5 or batch or fuzz or tile or small or golden" 2>&1 | tail -4 > gpurun_out/r11_gpu_suite.txt
for f in 0 1; do
  echo "fam $f base: $(abl/tile_probe_base 65536 128 128 $f | tail -2 | tr '\n' ' ')" >> gpurun_out/r11_phases.txt
  echo "fam $f new : $(tools/tile_probe 65536 128 128 $f | tail -2 | tr '\n' ' ')" >> gpurun_out/r11_phases.txt
done
cp paper_1707_05062_b200/lib/libkohler_cuda.so /tmp/cur.so
for v in base k5c base k5c; do cp abl/$v.so paper_1707_05062_b200/lib/libkohler_cuda.so; echo "$v $(python tools/ab_time.py --configs C5 2>&1 | tail -1)" >> gpurun_out/r11_ab.txt; done
cp /tmp/cur.so paper_1707_05062_b200/lib/libkohler_cuda.so
cat gpurun_out/r11_gpu_suite.txt gpurun_out/r11_phases.txt gpurun_out/r11_ab.txt
