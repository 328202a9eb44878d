# HEAD: tests, smoke, C2 line, reference arm; friendster-shaped single-GPU
# run refreshed with the current kernels.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 400 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2>/dev/null; cat gpurun_out/bench_c2.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>/dev/null; cat gpurun_out/bench_ref.json
SCALE=27 SAMPLES=1900000000 timeout 1500 python scripts/big_graph.py > gpurun_out/big27.jsonl 2>&1; echo rc $?; tail -14 gpurun_out/big27.jsonl | cut -c1-300
