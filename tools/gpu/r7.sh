# ncu --set full with source of K5 (C5) and K1 (C4): where do the shared-atomic "bank conflicts" come from?
cd $GRAFT_REPO_ROOT
timeout 120 python tools/run_config.py --config C5 --reps 2 > /dev/null 2>&1 && \
timeout 500 ncu --set full --import-source on --clock-control none -k regex:twalk_kernel -s 1 -c 1 -o gpurun_out/r7_c5_twalk python tools/run_config.py --config C5 --reps 2 > gpurun_out/r7_ncu_c5.log 2>&1
timeout 500 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 3 -c 1 -o gpurun_out/r7_c4_walk python tools/run_config.py --config C4 --reps 5 > gpurun_out/r7_ncu_c4.log 2>&1
ls -la gpurun_out
