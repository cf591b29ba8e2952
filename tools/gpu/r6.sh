# atomic-pattern probe (timing + ncu conflict counters) and a baseline A/B timing of the current build
set -u
tools/atom_probe > gpurun_out/r6_atom_probe.jsonl 2>&1
ncu --metrics smsp__inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,gpu__time_duration.sum --clock-control none --csv tools/atom_probe > gpurun_out/r6_atom_probe_ncu.csv 2>&1
python tools/ab_time.py --configs C1,C2,C3,C4,C5 > gpurun_out/r6_ab_base.txt 2>&1
cat gpurun_out/r6_atom_probe.jsonl gpurun_out/r6_ab_base.txt
