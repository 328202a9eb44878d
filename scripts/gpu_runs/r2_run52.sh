# round 2, run 52: per-round lr decay in the tournament -- tests, C3 (vertex
# and edge-scaled) and C4 sharded AUCROC, C1 sharded parity (30 seeds)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tournament.py tests/test_config_scale.py -q -m gpu -k "not c4_shape and not coarsening_matches" > gpurun_out/r2_52_tests.txt 2>&1
UNIT=vertex-pass RANKS=8 SHARD=1,2,3 timeout 900 python scripts/c3_shard_levels.py > gpurun_out/r2_52_c3_shard_vertex.jsonl 2>&1
UNIT=edge-scaled RANKS=8 SHARD=1,2,3 timeout 1200 python scripts/c3_shard_levels.py > gpurun_out/r2_52_c3_shard_edge.jsonl 2>&1
RANKS=2,4,8 timeout 1500 python scripts/c1_sharded_auc.py > gpurun_out/r2_52_c1_sharded.jsonl 2>&1
timeout 1200 python scripts/c4_sharded.py > gpurun_out/r2_52_c4_sharded.jsonl 2>&1
