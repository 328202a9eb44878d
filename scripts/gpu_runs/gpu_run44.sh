# Occupancy experiments on C2 and the tournament: 3 blocks/SM build (80 regs,
# spills), 16 lanes per source; tournament at d=256 (C5 dimension).
mkdir -p gpurun_out
for env in "X=0" "GB_LIB_PATH=build/exp/libgosh_b200_minb3.so" "GB_GROUP_LANES=16"; do
  echo "== c2 $env"
  env $env timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['roofline']['frac'])"
  echo "== tournament $env"
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
done
timeout 300 python bench.py --workload tournament --dim 256 --steps 10 --warmup 3 > gpurun_out/tourn_d256.json 2>/dev/null; cat gpurun_out/tourn_d256.json
GB_GROUP_LANES=8 timeout 300 python bench.py --workload tournament --dim 256 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('d256 G8', d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
ls gpurun_out
