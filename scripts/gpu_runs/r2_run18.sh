# round 2, run 18: pinned numpy sources take the direct DMA; e2e phases, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_io.py -q -m gpu -k staged > gpurun_out/r2_18_tests.txt 2>&1
timeout 600 python scripts/profile_multilevel_e2e.py > gpurun_out/r2_18_e2e_phases.jsonl 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_18_bench.json 2> gpurun_out/r2_18_bench.err
