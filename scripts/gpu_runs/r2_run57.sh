# round 2, run 57: row-gather probe with TMA bulk copies and bulk reduce-adds
mkdir -p gpurun_out build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/probe_rows scripts/probe_row_bandwidth.cu
for i in 1 2; do timeout 300 build/probe_rows; done > gpurun_out/r2_57_probe_rows.jsonl 2>&1
