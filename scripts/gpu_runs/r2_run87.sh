# round 2, run 87: one-shot coarse-CSR workspace kept across levels -- GPU
# coarsening tests, C4-shape e2e with phases
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_config_scale.py -q -m gpu -x > gpurun_out/r2_87_pytest.txt 2>&1
timeout 1500 python scripts/c4_e2e.py > gpurun_out/r2_87_c4_e2e.jsonl 2> gpurun_out/r2_87.err
