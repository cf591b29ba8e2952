set -x
cd $GRAFT_REPO_ROOT
timeout 60 tools/phase_probe > gpurun_out/phase_c2.txt 2>&1
timeout 60 tools/phase_probe 16384 16384 > gpurun_out/phase_c4.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 30 --warmup 5 > gpurun_out/ncu_launch.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 30 -c 1 -o gpurun_out/c2_walk python bench.py --steps 40 --warmup 5 > gpurun_out/ncu_c2.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 3 -c 1 -o gpurun_out/c4_walk python tools/run_config.py --config C4 --reps 5 > gpurun_out/ncu_c4.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:twalk_kernel -s 2 -c 1 -o gpurun_out/c5_twalk python tools/run_config.py --config C5 --reps 4 > gpurun_out/ncu_c5.log 2>&1
ls -la gpurun_out
