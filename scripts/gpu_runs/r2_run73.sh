# round 2, run 73: column-form row blocks (segmented sort of 32-bit columns)
# -- parity tests, C5 coarsening phases in both forms, C5 end to end
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_config_scale.py -q -m gpu -x -k "blocked or c5_path or csr_from" > gpurun_out/r2_73_pytest.txt 2>&1
GB_TRACE_BLOCKS=1 SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_73_c5_cols.jsonl 2> gpurun_out/r2_73.err
GB_COARSE_BLOCK_FORM=keys GB_TRACE_BLOCKS=1 SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_73_c5_keys.jsonl 2>> gpurun_out/r2_73.err
timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_73_c5_multilevel.jsonl 2>> gpurun_out/r2_73.err
