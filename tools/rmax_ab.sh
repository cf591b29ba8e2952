# A/B of the longest column walk the launcher may pick (KOHLER_RMAX, rows
# per walk): bench C2 line, C3 / C4 device timings, and the parity suites at
# the longest setting.  Run from the repo root on the GPU box.
cd $GRAFT_REPO_ROOT
for r in 64 96 128; do
    v=$(KOHLER_RMAX=$r timeout 300 python bench.py 2>&1 | tail -1 | cut -c 100-200)
    echo "R$r bench $v"
    for c in C3 C4; do
        v=$(KOHLER_RMAX=$r timeout 120 python tools/run_config.py --config $c --time 2>&1 | tail -1 | cut -c 120-220)
        echo "R$r $c $v"
    done
done
KOHLER_RMAX=128 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
