# round 2, run 79: rotation-mean lr (GB_ROUND_LR=rotation_mean) vs per-round
# decay on the sharded AUCROC regimes: C4 10 edge-scaled epochs (the
# one-rotation extreme), C4 CLI vertex-pass, C3 edge-scaled and vertex-pass
mkdir -p gpurun_out
for mode in round rotation_mean; do
GB_ROUND_LR=$mode UNIT=edge-scaled EPOCHS=10 SHARD=1,2 timeout 1500 python scripts/c4_sharded.py > gpurun_out/r2_79_c4_es10_$mode.jsonl 2>> gpurun_out/r2_79.err
GB_ROUND_LR=$mode UNIT=vertex-pass EPOCHS=1000 SHARD=1,2 timeout 900 python scripts/c3_shard_levels.py > gpurun_out/r2_79_c3_vp_$mode.jsonl 2>> gpurun_out/r2_79.err
done
