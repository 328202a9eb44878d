mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --workload tournament --steps 3 --warmup 3 > gpurun_out/bench_tour.json 2> gpurun_out/bench_tour.err; tail -3 gpurun_out/bench_tour.err; cat gpurun_out/bench_tour.json
RANKS=0,1,2,4 SEEDS=1,2,3 timeout 900 python scripts/sharded_auc.py c1 > gpurun_out/sharded_auc_c1.jsonl 2> gpurun_out/sharded_auc_c1.err; tail -3 gpurun_out/sharded_auc_c1.err; cat gpurun_out/sharded_auc_c1.jsonl
UNIT=vertex-pass timeout 900 python scripts/bench_multilevel.py c3 1000 > gpurun_out/ml_c3_vp.jsonl 2> gpurun_out/ml_c3_vp.err; tail -3 gpurun_out/ml_c3_vp.err; cat gpurun_out/ml_c3_vp.jsonl
UNIT=edge-scaled timeout 1200 python scripts/bench_multilevel.py c3 1000 > gpurun_out/ml_c3_es.jsonl 2> gpurun_out/ml_c3_es.err; tail -3 gpurun_out/ml_c3_es.err; cat gpurun_out/ml_c3_es.jsonl
