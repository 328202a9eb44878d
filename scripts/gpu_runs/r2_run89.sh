# round 2, run 89: the C4-shape end-to-end embed under torch's native caching
# allocator instead of cudaMallocAsync (twice)
mkdir -p gpurun_out
for i in 1 2; do PYTORCH_CUDA_ALLOC_CONF=backend:native REPS=2 timeout 1500 python scripts/c4_e2e.py > gpurun_out/r2_89_c4_e2e_native_$i.jsonl 2>> gpurun_out/r2_89.err; done
