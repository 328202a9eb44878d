# Pair kernel: L2 bulk prefetch of the next sample window (A/B) + tests + ncu.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for env in "GB_POOL_PREFETCH=0" "GB_POOL_PREFETCH=1"; do
  echo "== tournament $env"
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_pool_kernel -s 6 -c 1 -o gpurun_out/pool_pf python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1
ls gpurun_out
