mkdir -p gpurun_out
for pipe in 0 1; do
GB_PIPE=$pipe CAPS=0,16,64 SEEDS=1,2,3 timeout 900 python scripts/c1_gpu_auc.py > gpurun_out/c1auc_pipe$pipe.jsonl 2>gpurun_out/c1auc_pipe$pipe.err; tail -2 gpurun_out/c1auc_pipe$pipe.err; cat gpurun_out/c1auc_pipe$pipe.jsonl
done
DETERMINISTIC=1 CAPS=0 SEEDS=1 timeout 1200 python scripts/c1_gpu_auc.py > gpurun_out/c1auc_det.jsonl 2>gpurun_out/c1auc_det.err; tail -2 gpurun_out/c1auc_det.err; cat gpurun_out/c1auc_det.jsonl
