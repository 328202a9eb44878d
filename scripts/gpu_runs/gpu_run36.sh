# Pair kernel: HOT kernels without the fused-pool code; lanes per source A/B.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for env in "GB_GROUP_LANES=8" "GB_GROUP_LANES=16" "GB_GROUP_LANES=32" "GB_GROUP_LANES=16 GB_POOL_PREFETCH=0" "GB_GROUP_LANES=8 GB_POOL_PREFETCH=0"; do
  echo "== tournament $env"
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
done
ls gpurun_out
