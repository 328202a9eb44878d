# round 2, run 90: C5 end to end under torch's native caching allocator (twice)
mkdir -p gpurun_out
for i in 1 2; do PYTORCH_CUDA_ALLOC_CONF=backend:native timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_90_c5_native_$i.jsonl 2>> gpurun_out/r2_90.err; done
