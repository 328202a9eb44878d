mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 900 python scripts/bench_large.py > gpurun_out/large22.jsonl 2>&1; tail -1 gpurun_out/large22.jsonl
SCALE=24 SAMPLES=250000000 BUDGET_GB=3 timeout 1200 python scripts/bench_large.py > gpurun_out/large24.jsonl 2>&1; tail -2 gpurun_out/large24.jsonl
