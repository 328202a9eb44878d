# round 2, run 77: R-MAT samples kept across row blocks -- parity tests, C5 end to end
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_config_scale.py -q -m gpu -x -k "blocked or c5_path or csr_from" > gpurun_out/r2_77_pytest.txt 2>&1
for i in 1 2; do timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_77_c5_$i.jsonl 2>> gpurun_out/r2_77.err; done
