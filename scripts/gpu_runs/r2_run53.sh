# round 2, run 53: per-round lr decay with ONE sharded level: C1 parity (30
# seeds, 2/4/8 ranks), C4 edge-scaled, C3 vertex-pass seeds 2-3
mkdir -p gpurun_out
SHARD=1 RANKS=2,4,8 timeout 1500 python scripts/c1_sharded_auc.py > gpurun_out/r2_53_c1_sharded1.jsonl 2>&1
UNIT=edge-scaled EPOCHS=10 SHARD=1,2 timeout 1200 python scripts/c4_sharded.py > gpurun_out/r2_53_c4_sharded_edge.jsonl 2>&1
