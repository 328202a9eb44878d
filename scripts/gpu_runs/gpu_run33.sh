# Pair kernel: lane-parallel sample windows, compacted pools (gb_fill_pool_compact
# + gb_train_pool_list), forwarding behind a branch.  Tests + A/B + ncu.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -8
for env in "GB_POOL_MODE=fused" "GB_POOL_MODE=materialize" "GB_POOL_MODE=compact"; do
  echo "== tournament $env"
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
done
echo "== c2"
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['roofline']['frac'], d['e2e']['value']/1e9)"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/tourn_launches_compact.csv python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_pool_kernel -s 5 -c 1 -o gpurun_out/pool_list python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1
ls gpurun_out
