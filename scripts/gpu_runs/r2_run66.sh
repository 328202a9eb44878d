# round 2, run 66: per-row key cursors in the row-block coarse CSR -- parity
# tests, then the C5-shape coarsening phases again
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_config_scale.py -q -m gpu -x -k "blocked or c5_path or csr_from" > gpurun_out/r2_66_pytest.txt 2>&1
SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_66_coarsen_c5.jsonl 2> gpurun_out/r2_66.err
