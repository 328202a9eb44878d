# round 2, run 68: where csr_from_blocks' setup time goes at the C5 shape, with
# the default mempool's release threshold as torch leaves it and at max
mkdir -p gpurun_out
GB_TRACE_BLOCKS=1 SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_68_c5_default.jsonl 2> gpurun_out/r2_68.err
RELEASE=1 GB_TRACE_BLOCKS=1 SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_68_c5_release_max.jsonl 2>> gpurun_out/r2_68.err
