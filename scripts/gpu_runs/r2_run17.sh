# round 2, run 17: threaded pinned staging -- tests, C3 e2e phases, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_io.py tests/test_gpu_parity.py tests/test_ppr.py -q -m gpu > gpurun_out/r2_17_tests.txt 2>&1
timeout 600 python scripts/profile_multilevel_e2e.py > gpurun_out/r2_17_e2e_phases.jsonl 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_17_bench.json 2> gpurun_out/r2_17_bench.err
