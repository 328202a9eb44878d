# Pair kernel with the next chunk cp.async-staged in shared memory while the
# current chunk trains from registers (GB_POOL_PIPE=1): tests under it, A/B.
mkdir -p gpurun_out
GB_POOL_PIPE=1 timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for env in "GB_POOL_PIPE=0" "GB_POOL_PIPE=1" "GB_POOL_PIPE=0" "GB_POOL_PIPE=1"; do
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env d128', d['value']/1e9, d['roofline']['frac'])"
  env $env timeout 300 python bench.py --workload tournament --dim 256 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env d256', d['value']/1e9, d['roofline']['frac'])"
done
