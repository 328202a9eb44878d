mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/bench1.json 2>gpurun_out/bench1.err; tail -2 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 300 python bench.py --workload tournament --steps 3 --warmup 3 > gpurun_out/bench_tour.json 2>&1; tail -1 gpurun_out/bench_tour.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_tour.csv python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu1 $?
CAPS=0 SEEDS=1,2,3,4,5 timeout 900 python scripts/c1_gpu_auc.py > gpurun_out/c1auc_default.jsonl 2>gpurun_out/c1auc_default.err; tail -2 gpurun_out/c1auc_default.err; cat gpurun_out/c1auc_default.jsonl
CPU=1 UNIT=vertex-pass timeout 1200 python scripts/bench_multilevel.py c3 1000 > gpurun_out/ml_c3_vp.jsonl 2> gpurun_out/ml_c3_vp.err; tail -3 gpurun_out/ml_c3_vp.err; cat gpurun_out/ml_c3_vp.jsonl
UNIT=edge-scaled timeout 1200 python scripts/bench_multilevel.py c3 1000 > gpurun_out/ml_c3_es.jsonl 2> gpurun_out/ml_c3_es.err; tail -3 gpurun_out/ml_c3_es.err; cat gpurun_out/ml_c3_es.jsonl
