# round 2, run 91: C5 and C4-shape end to end under the native allocator with
# expandable segments
mkdir -p gpurun_out
for i in 1 2; do PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_91_c5_exp_$i.jsonl 2>> gpurun_out/r2_91.err; done
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True REPS=2 timeout 1500 python scripts/c4_e2e.py > gpurun_out/r2_91_c4_exp.jsonl 2>> gpurun_out/r2_91.err
