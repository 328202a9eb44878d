# round 2, run 64: coarsening phase breakdown at the C5 shape (row-block builds)
mkdir -p gpurun_out
SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_64_coarsen_c5.jsonl 2> gpurun_out/r2_64.err
