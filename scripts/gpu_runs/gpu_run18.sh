mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
SCALE=24 SAMPLES=500000000 timeout 900 python scripts/big_graph.py > gpurun_out/big24.jsonl 2>&1; echo rc $?; cat gpurun_out/big24.jsonl | tail -12
SCALE=26 SAMPLES=2000000000 timeout 1500 python scripts/big_graph.py > gpurun_out/big26.jsonl 2>&1; echo rc $?; cat gpurun_out/big26.jsonl | tail -14
