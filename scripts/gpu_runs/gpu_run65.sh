# AUCROC at HEAD (staged pass default for uncapped launches): C1 5 seeds,
# C3 vertex-pass 100 epochs in-memory (2 seeds) + balanced tournament K=16.
mkdir -p gpurun_out
CAPS=0 SEEDS=1,2,3,4,5 timeout 900 python scripts/c1_gpu_auc.py > gpurun_out/c1auc.jsonl 2>/dev/null; cut -c1-200 gpurun_out/c1auc.jsonl
GRAPH=c3 MODES=cap0,tour8b SEEDS=1,2 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000 timeout 1500 python scripts/auc_modes.py > gpurun_out/c3_auc_head.jsonl 2>/dev/null; cut -c1-200 gpurun_out/c3_auc_head.jsonl
