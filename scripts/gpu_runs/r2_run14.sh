# round 2, run 14: full GPU suite (PPR, C4-shape checksum test, cached
# graphs), smoke, the default bench line + reference arm, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_14_gpu.txt
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_14_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_14_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_14_bench.json 2> gpurun_out/r2_14_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_14_bench_ref.json 2> gpurun_out/r2_14_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_14_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_14_ncu_bench.log 2>&1
