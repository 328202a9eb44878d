# Pair kernel after cleanup: tests, tournament K=2 and K=16 (8 virtual ranks),
# launch list + ncu of the off-diagonal pair kernel, C1 sharded AUCROC.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 > gpurun_out/tourn_k2.json 2>/dev/null; cat gpurun_out/tourn_k2.json
timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 3 --warmup 3 > gpurun_out/tourn_k16.json 2>/dev/null; cat gpurun_out/tourn_k16.json
GB_POOL_MODE=fused timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fused k16', d['value']/1e9, d['roofline']['frac'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/tourn_launches_k2.csv python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:train_pool_kernel.*Li1EE -s 2 -c 1 -o gpurun_out/pool_offdiag python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1
RANKS=0,1,2,4 SEEDS=1,2,3 timeout 900 python scripts/sharded_auc.py c1 > gpurun_out/sharded_auc_c1.jsonl 2>/dev/null; cat gpurun_out/sharded_auc_c1.jsonl | cut -c1-200
ls gpurun_out
