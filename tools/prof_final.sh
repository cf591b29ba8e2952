# Final capture of the shipped configuration (run from the repo root on the
# GPU box): launch list of a short bench run and ncu --set full of K1 on a C2
# bench step and on C4; each ncu command after the same command exited 0.
cd $GRAFT_REPO_ROOT
timeout 120 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_short.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 30 --warmup 5 > gpurun_out/ncu_launch.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 30 -c 1 -o gpurun_out/c2_walk python bench.py --steps 40 --warmup 5 > gpurun_out/ncu_c2.log 2>&1
timeout 120 python tools/run_config.py --config C4 --reps 5 > /dev/null 2>&1 && \
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 3 -c 1 -o gpurun_out/c4_walk python tools/run_config.py --config C4 --reps 5 > gpurun_out/ncu_c4.log 2>&1
ls gpurun_out
