mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
GRAPH=c1 MODES=cap0 SEEDS=1,1,1,1,1,2,3,4,5 timeout 900 python scripts/auc_modes.py > gpurun_out/auc_c1_rep.jsonl 2> gpurun_out/auc_c1_rep.err; tail -3 gpurun_out/auc_c1_rep.err; cat gpurun_out/auc_c1_rep.jsonl
GRAPH=c3 MODES=cap0,det SEEDS=1 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000 timeout 1500 python scripts/auc_modes.py > gpurun_out/auc_c3.jsonl 2> gpurun_out/auc_c3.err; tail -3 gpurun_out/auc_c3.err; cat gpurun_out/auc_c3.jsonl
