# round 2, run 92: final HEAD validation -- GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_92_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_92_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2_92_bench.json 2> gpurun_out/r2_92_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2_92_bench_ref.json 2> gpurun_out/r2_92_bench_ref.err
