mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python bench.py --workload tournament --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-200
SCALE=27 SAMPLES=1900000000 timeout 1500 python scripts/big_graph.py > gpurun_out/big27c.jsonl 2>&1; echo rc $?; cut -c1-300 gpurun_out/big27c.jsonl | tail -12
