mkdir -p gpurun_out
free -g | head -2; nproc
SCALE=27 SAMPLES=1900000000 timeout 1500 python scripts/big_graph.py > gpurun_out/big27.jsonl 2>&1; echo rc $?; tail -12 gpurun_out/big27.jsonl | cut -c1-600
