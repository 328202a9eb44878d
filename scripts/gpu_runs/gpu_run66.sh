# C5 path on one GPU at HEAD: train_large with the matrix in pinned host
# memory (compacted pools + HOT pair kernel now), R-MAT scale 24, d=256.
mkdir -p gpurun_out
SCALE=24 SAMPLES=250000000 BUDGET_GB=3 timeout 1200 python scripts/bench_large.py > gpurun_out/large24.jsonl 2>&1; tail -2 gpurun_out/large24.jsonl | cut -c1-500
