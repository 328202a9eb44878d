mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_store.json 2>gpurun_out/bench_store.err; tail -2 gpurun_out/bench_store.err; cat gpurun_out/bench_store.json
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --atomic-rows > gpurun_out/bench_atomic.json 2>gpurun_out/bench_atomic.err; tail -2 gpurun_out/bench_atomic.err; cat gpurun_out/bench_atomic.json
timeout 300 python bench.py --workload tournament --steps 3 --warmup 3 --atomic-rows > gpurun_out/bench_tour_atomic.json 2>&1; tail -1 gpurun_out/bench_tour_atomic.json
GRAPH=c1 MODES=cap0a SEEDS=1,1,1,2,3,4,5 timeout 900 python scripts/auc_modes.py > gpurun_out/auc_c1_atomic.jsonl 2> gpurun_out/auc_c1_atomic.err; tail -3 gpurun_out/auc_c1_atomic.err; cat gpurun_out/auc_c1_atomic.jsonl
GRAPH=c3 MODES=cap0a,cap0 SEEDS=1,2 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000 timeout 1500 python scripts/auc_modes.py > gpurun_out/auc_c3_atomic.jsonl 2> gpurun_out/auc_c3_atomic.err; tail -3 gpurun_out/auc_c3_atomic.err; cat gpurun_out/auc_c3_atomic.jsonl
