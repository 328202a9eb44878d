# C3 edge-scaled AUCROC of the reference's partitioned algorithm on one GPU
# (train_large, K = 8 / 16) -- the baseline the tournament (tour4 / tour8) shards.
mkdir -p gpurun_out
GRAPH=c3 MODES=large8,large16 SEEDS=1 UNIT=edge-scaled EPOCHS=1000 EVAL_SAMPLE=1000000 timeout 2400 python scripts/auc_modes.py > gpurun_out/c3_auc_large_es.jsonl 2> gpurun_out/c3_auc_large_es.err; tail -3 gpurun_out/c3_auc_large_es.err; cut -c1-300 gpurun_out/c3_auc_large_es.jsonl
