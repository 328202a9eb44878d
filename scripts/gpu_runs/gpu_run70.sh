mkdir -p gpurun_out
for vs in 0 1; do
GB_VIRTUAL_STREAMS=$vs RANKS=4,8 SEEDS=1,2,3 timeout 900 python scripts/sharded_auc.py c1 > gpurun_out/sharded_auc_c1_vs$vs.jsonl 2> gpurun_out/sharded_auc_c1_vs$vs.err; tail -2 gpurun_out/sharded_auc_c1_vs$vs.err; echo "vs=$vs"; cat gpurun_out/sharded_auc_c1_vs$vs.jsonl
done
