# round 2, run 83: hubs split over all warps in the row-block key appends --
# parity tests (incl. a 32-arc threshold), C5 coarsening phases, C5 end to end
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_config_scale.py -q -m gpu -x -k "blocked or c5_path or csr_from" > gpurun_out/r2_83_pytest.txt 2>&1
GB_TRACE_BLOCKS=1 SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_83_c5_phases.jsonl 2> gpurun_out/r2_83.err
timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_83_c5_multilevel.jsonl 2>> gpurun_out/r2_83.err
