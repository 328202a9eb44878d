# round 2, run 80: a sub-rotation budget as several rotations of B=1 instead
# of one rotation of B=round(eff/K) (GB_SUBROTATION_BATCH=1, experiment): C4
# shape, 10 edge-scaled epochs, 8 ranks
mkdir -p gpurun_out
GB_SUBROTATION_BATCH=1 UNIT=edge-scaled EPOCHS=10 SHARD=1,2 timeout 1500 python scripts/c4_sharded.py > gpurun_out/r2_80_c4_es10_b1.jsonl 2> gpurun_out/r2_80.err
