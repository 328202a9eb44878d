# round 2, run 19: full GPU suite + smoke + bench at HEAD (PassArgs layout fix)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_19_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_19_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_19_bench.json 2> gpurun_out/r2_19_bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-multilevel > gpurun_out/r2_19_bench2.json 2> gpurun_out/r2_19_bench2.err
