# round 2, run 100: final HEAD validation (device pair subsample) -- GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_100_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_100_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2_100_bench.json 2> gpurun_out/r2_100_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2_100_bench_ref.json 2> gpurun_out/r2_100_bench_ref.err
