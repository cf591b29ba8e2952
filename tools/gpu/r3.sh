python -m pytest tests/test_acceptance_relink.py -q -s 2>&1 | tail -40 > gpurun_out/r3_acceptance.txt
cat gpurun_out/r3_acceptance.txt
