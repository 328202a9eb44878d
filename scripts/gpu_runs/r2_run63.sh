# round 2, run 63: coarsening phase breakdown at the C4 (friendster) shape
mkdir -p gpurun_out
SCALE=27 SAMPLES=1900000000 timeout 900 python scripts/profile_coarsen.py > gpurun_out/r2_63_coarsen_c4.jsonl 2> gpurun_out/r2_63.err
