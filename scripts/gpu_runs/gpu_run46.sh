# C3 AUCROC: in-memory Hogwild vs the sharded multilevel path (finest levels by
# the part-pair tournament over 1/4/8 virtual ranks = K 2/8/16), vertex-pass
# 100 epochs, 1M+1M eval sample; reference-equivalent (deterministic) 0.7053.
mkdir -p gpurun_out
GRAPH=c3 MODES=cap0,tour1,tour4,tour8 SEEDS=1,2 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000 timeout 2400 python scripts/auc_modes.py > gpurun_out/c3_auc_tour.jsonl 2> gpurun_out/c3_auc_tour.err; tail -2 gpurun_out/c3_auc_tour.err; cut -c1-300 gpurun_out/c3_auc_tour.jsonl
