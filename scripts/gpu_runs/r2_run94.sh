# round 2, run 94: the native allocator with max_split_size_mb=1024 (large
# cached blocks are never split) -- C5 end to end, C4-shape end to end
mkdir -p gpurun_out
PYTORCH_CUDA_ALLOC_CONF=max_split_size_mb:1024 timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_94_c5_nosplit.jsonl 2>> gpurun_out/r2_94.err
PYTORCH_CUDA_ALLOC_CONF=max_split_size_mb:1024 REPS=2 timeout 1500 python scripts/c4_e2e.py > gpurun_out/r2_94_c4_nosplit.jsonl 2>> gpurun_out/r2_94.err
