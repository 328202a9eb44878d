mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --workload tournament --steps 3 --warmup 3 --atomic-rows > gpurun_out/bench_tour_atomic2.json 2>&1; tail -1 gpurun_out/bench_tour_atomic2.json
GRAPH=c3 MODES=cap256a,cap1024a SEEDS=1 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000 timeout 900 python scripts/auc_modes.py > gpurun_out/auc_c3_caps_a.jsonl 2>&1; cat gpurun_out/auc_c3_caps_a.jsonl | grep mode
GB_PIPE=0 GRAPH=c3 MODES=cap256,cap256a SEEDS=1 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000 timeout 900 python scripts/auc_modes.py > gpurun_out/auc_c3_caps_nopipe.jsonl 2>&1; cat gpurun_out/auc_c3_caps_nopipe.jsonl | grep mode
for fl in 8 16 32; do
GB_INFLIGHT_FLOOR=$fl GRAPH=c1 MODES=cap0a SEEDS=1,2,3,4,5 timeout 900 python scripts/auc_modes.py > gpurun_out/auc_c1_floor$fl.jsonl 2>&1; echo floor $fl; grep mode gpurun_out/auc_c1_floor$fl.jsonl
done
