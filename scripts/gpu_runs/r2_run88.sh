# round 2, run 88: host-side copy threads of the staged transfers (8 vs 16)
# on the C4-shape end-to-end embed; the box's core count
mkdir -p gpurun_out
nproc > gpurun_out/r2_88_nproc.txt
for n in 8 16; do GB_STAGING_THREADS=$n REPS=2 timeout 1500 python scripts/c4_e2e.py > gpurun_out/r2_88_c4_e2e_t$n.jsonl 2>> gpurun_out/r2_88.err; done
