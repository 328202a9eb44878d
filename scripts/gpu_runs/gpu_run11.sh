mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches_tour.csv python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu1 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_pool -s 6 -c 1 -o gpurun_out/prof_pool python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu2 $?
for div in 64 16 4 1; do
GB_INFLIGHT_DIV=$div GRAPH=c1 MODES=cap0 SEEDS=1,2,3,4,5 timeout 900 python scripts/auc_modes.py > gpurun_out/auc_c1_div$div.jsonl 2> gpurun_out/auc_c1_div$div.err; tail -2 gpurun_out/auc_c1_div$div.err; cat gpurun_out/auc_c1_div$div.jsonl
done
GRAPH=c3 MODES=cap0,cap4096,cap1024,cap256 SEEDS=1,2 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000 timeout 1500 python scripts/auc_modes.py > gpurun_out/auc_c3_caps.jsonl 2> gpurun_out/auc_c3_caps.err; tail -3 gpurun_out/auc_c3_caps.err; cat gpurun_out/auc_c3_caps.jsonl
