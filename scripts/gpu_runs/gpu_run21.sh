mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -4
SCALE=27 SAMPLES=1900000000 timeout 1500 python scripts/big_graph.py > gpurun_out/big27b.jsonl 2>&1; echo rc $?; head -3 gpurun_out/big27b.jsonl | cut -c1-300; tail -1 gpurun_out/big27b.jsonl
