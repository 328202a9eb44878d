# Final HEAD check after dropping the staged-pair experiment: tests, smoke,
# C2 line + reference arm, tournament line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2>/dev/null; cut -c1-120 gpurun_out/bench_c2.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>/dev/null; cut -c1-120 gpurun_out/bench_ref.json
timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 > gpurun_out/tourn_k2.json 2>/dev/null; cut -c1-120 gpurun_out/tourn_k2.json
