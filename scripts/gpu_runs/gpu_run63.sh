# Experiment: pair kernel with the sample rows staged in shared memory
# (-DGB_POOL_STAGED build): GPU tests under it, tournament A/B d=128/256.
mkdir -p gpurun_out
GB_LIB_PATH=build/exp/libgosh_b200_poolstaged.so timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for env in "X=0" "GB_LIB_PATH=build/exp/libgosh_b200_poolstaged.so" "X=0" "GB_LIB_PATH=build/exp/libgosh_b200_poolstaged.so"; do
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env d128', d['value']/1e9, d['roofline']['frac'])"
  env $env timeout 300 python bench.py --workload tournament --dim 256 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env d256', d['value']/1e9, d['roofline']['frac'])"
done
