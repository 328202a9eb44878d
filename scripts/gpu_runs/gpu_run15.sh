mkdir -p gpurun_out
for v in "" "--store-rows"; do
timeout 300 python bench.py --workload tournament --steps 3 --warmup 3 $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'])"
GB_INFLIGHT_DIV=8 timeout 300 python bench.py --workload tournament --steps 3 --warmup 3 $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('div8 $v', d['value'], d['ms_per_step'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_pool -s 6 -c 1 -o gpurun_out/prof_pool2 python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu2 $?
