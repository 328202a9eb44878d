# HOT kernel instantiations (compile-time default flags) and materialized
# pools: A/B on the tournament and the C2 pass, plus the GPU tests.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
for env in "GB_NO_HOT=1" "GB_NO_HOT=0" "GB_NO_HOT=1 GB_POOL_MATERIALIZE=1" "GB_NO_HOT=0 GB_POOL_MATERIALIZE=1"; do
  echo "== tournament $env"
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
done
for env in "GB_NO_HOT=1" "GB_NO_HOT=0"; do
  echo "== c2 $env"
  env $env timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['roofline']['frac'], d['e2e']['value']/1e9)"
done
GB_POOL_MATERIALIZE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/tourn_launches_mat.csv python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/tourn_launches.csv python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_pool_kernel -s 4 -c 1 -o gpurun_out/pool_hot python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1
ls gpurun_out
