# Final round-2 capture set (r02i_*), after the walk-length chooser change: full GPU suite, three bench lines at the
# driver's invocation, per-config timings, the launch list, ncu --set full of
# K1 (C2 bench step, C4), the cluster K1 (C1) and K5 (C5).  Each ncu command
# runs only after the same command exited 0 without ncu.
cd $GRAFT_REPO_ROOT
set -u
O=gpurun_out/r02i
mkdir -p $O
python -m pytest tests -q -m gpu 2>&1 | tail -4 > $O/gpu_suite.txt
for i in 1 2 3; do timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench_c2_run$i.json 2> $O/bench_run$i.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_ref.err
python tools/ab_time.py --configs C1,C2,C3,C4,C5 > $O/ab_configs.json 2>&1
timeout 120 python bench.py --steps 30 --warmup 5 --no-per-config > /dev/null 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2_bench.csv python bench.py --steps 30 --warmup 5 --no-per-config > $O/ncu_launch.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 30 -c 1 -o $O/c2_walk python bench.py --steps 40 --warmup 5 --no-per-config > $O/ncu_c2.log 2>&1
timeout 120 python tools/run_config.py --config C4 --reps 5 > /dev/null 2>&1 && \
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 3 -c 1 -o $O/c4_walk python tools/run_config.py --config C4 --reps 5 > $O/ncu_c4.log 2>&1
timeout 120 python tools/run_config.py --config C1 --reps 5 > /dev/null 2>&1 && \
timeout 400 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -s 5 -c 1 -o $O/c1_walk_cluster python tools/run_config.py --config C1 --reps 10 > $O/ncu_c1.log 2>&1
timeout 500 ncu --set full --import-source on --clock-control none -k regex:twalk_kernel -s 1 -c 1 -o $O/c5_twalk python tools/run_config.py --config C5 --reps 2 > $O/ncu_c5.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:select256 -s 1 -c 1 -o $O/c5_select256 python tools/run_config.py --config C5 --reps 2 > $O/ncu_c5_sel.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"twalk|select" -c 6 --csv --log-file $O/launches_c5.csv python tools/run_config.py --config C5 --reps 3 > $O/ncu_c5_launch.log 2>&1
tools/mix_probe > $O/mix_probe.jsonl 2>&1
ls -la $O
cat $O/gpu_suite.txt $O/ab_configs.json; for i in 1 2 3; do cut -c1-300 $O/bench_c2_run$i.json; done
