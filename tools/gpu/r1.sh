set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
for i in 1 2 3; do python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/b20_$i.json 2> gpurun_out/b20_$i.err; echo rc=$?; done
python bench.py --steps 500 --warmup 10 --no-per-config > gpurun_out/b500.json 2> gpurun_out/b500.err; echo rc=$?
tail -3 gpurun_out/*.err
