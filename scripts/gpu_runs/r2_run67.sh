# round 2, run 67: per-row cursors with strided vertex ownership; per-block trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_config_scale.py -q -m gpu -x -k "blocked or c5_path or csr_from" > gpurun_out/r2_67_pytest.txt 2>&1
GB_TRACE_BLOCKS=1 SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_67_coarsen_c5.jsonl 2> gpurun_out/r2_67.err
