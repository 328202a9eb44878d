# round 2, run 70: block key buffer + workspace reused across coarsening levels; parity tests;
# C5 end to end (build, coarsen, embed at d=256) on one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_config_scale.py -q -m gpu -x -k "blocked or c5_path or csr_from" > gpurun_out/r2_70_pytest.txt 2>&1
timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_70_c5_multilevel.jsonl 2> gpurun_out/r2_69.err
GB_TRACE_BLOCKS=1 SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_70_c5_phases.jsonl 2>> gpurun_out/r2_69.err
