# GPU tests; C1 sharded AUCROC with balanced pools (default of
# train_multilevel_sharded now) vs in-memory, 3 seeds.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
RANKS=0,1,2,4 SEEDS=1,2,3 timeout 900 python scripts/sharded_auc.py c1 > gpurun_out/sharded_auc_c1_bal.jsonl 2>/dev/null; cut -c1-220 gpurun_out/sharded_auc_c1_bal.jsonl
