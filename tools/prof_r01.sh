# One gpurun call that refreshes the round's evidence (run from the repo root
# on the GPU box): bench line, per-config timings, phase probes, the ncu
# launch list of a short bench run and ncu --set full captures of K1 (C2
# bench step, C4) and K5 (C5).  Every ncu command runs only after the same
# command exited 0 without ncu.
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
for c in C1 C3 C4 C5; do timeout 120 python tools/run_config.py --config $c --time 2>&1 | tail -1 >> gpurun_out/configs.log; done
timeout 120 python tools/run_config.py --config C2 --time --depth 1 2>&1 | tail -1 >> gpurun_out/configs.log
timeout 120 python tools/run_config.py --config C2 --time --depth 2 2>&1 | tail -1 >> gpurun_out/configs.log
for c in C2 C3 C4; do timeout 120 python tools/run_config.py --config $c --time --rgb 2>&1 | tail -1 >> gpurun_out/configs.log; done
for c in C3 C4; do KOHLER_RGB_UNFUSED=1 timeout 120 python tools/run_config.py --config $c --time --rgb 2>&1 | tail -1 >> gpurun_out/configs_rgb_two_pass.log; done
timeout 60 tools/phase_probe > gpurun_out/phase_c2.txt 2>&1
timeout 60 tools/phase_probe 16384 16384 > gpurun_out/phase_c4.txt 2>&1
timeout 120 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_short.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 30 --warmup 5 > gpurun_out/ncu_launch.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 30 -c 1 -o gpurun_out/c2_walk python bench.py --steps 40 --warmup 5 > gpurun_out/ncu_c2.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 3 -c 1 -o gpurun_out/c4_walk python tools/run_config.py --config C4 --reps 5 > gpurun_out/ncu_c4.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:twalk_kernel -s 2 -c 1 -o gpurun_out/c5_twalk python tools/run_config.py --config C5 --reps 4 > gpurun_out/ncu_c5.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 3 -c 1 -o gpurun_out/c4_rgb_walk python tools/run_config.py --config C4 --reps 5 --rgb > gpurun_out/ncu_c4rgb.log 2>&1
ls -la gpurun_out
