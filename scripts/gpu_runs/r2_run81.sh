# round 2, run 81: tournament lr per in-memory epoch (round_lr with the
# level's epochs) -- tournament GPU tests, then the sharded AUCROC regimes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tournament.py tests/test_config_scale.py -q -m gpu -x > gpurun_out/r2_81_pytest.txt 2>&1
UNIT=edge-scaled EPOCHS=10 SHARD=1,2 timeout 1500 python scripts/c4_sharded.py > gpurun_out/r2_81_c4_es10.jsonl 2>> gpurun_out/r2_81.err
UNIT=vertex-pass EPOCHS=200 SHARD=1,2 timeout 1500 python scripts/c4_sharded.py > gpurun_out/r2_81_c4_vp200.jsonl 2>> gpurun_out/r2_81.err
UNIT=vertex-pass EPOCHS=1000 SHARD=1,2 timeout 900 python scripts/c3_shard_levels.py > gpurun_out/r2_81_c3_vp.jsonl 2>> gpurun_out/r2_81.err
UNIT=edge-scaled EPOCHS=1000 SHARD=1 timeout 1500 python scripts/c3_shard_levels.py > gpurun_out/r2_81_c3_es.jsonl 2>> gpurun_out/r2_81.err
RANKS=2,4 SHARD=1 NSEEDS=30 timeout 1800 python scripts/c1_sharded_auc.py > gpurun_out/r2_81_c1.jsonl 2>> gpurun_out/r2_81.err
