# round 2, run 99: evaluation positives subsampled from the device pair
# enumeration -- eval GPU tests, C4-shape setup phases
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_eval.py tests/test_integration.py -q -m gpu -x > gpurun_out/r2_99_pytest.txt 2>&1
timeout 1200 python scripts/c4_setup_phases.py > gpurun_out/r2_99_c4_setup.jsonl 2> gpurun_out/r2_99.err
