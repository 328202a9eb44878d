# Experiment: rolling gathers with a one-sample refill delay (-DGB_POOL_ROLL
# build) -- GPU tests under it, tournament A/B at d=128 and d=256.
mkdir -p gpurun_out
GB_LIB_PATH=build/exp/libgosh_b200_roll.so timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for env in "X=0" "GB_LIB_PATH=build/exp/libgosh_b200_roll.so" "X=0" "GB_LIB_PATH=build/exp/libgosh_b200_roll.so"; do
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env d128', d['value']/1e9, d['roofline']['frac'])"
  env $env timeout 300 python bench.py --workload tournament --dim 256 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env d256', d['value']/1e9, d['roofline']['frac'])"
done
