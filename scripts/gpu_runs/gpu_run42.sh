# Pair kernel with rolling gathers (slot refilled right after its update);
# C2 pass KIND 2 (index chain one ahead) default.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for w in "--virtual-ranks 1 --steps 10" "--virtual-ranks 1 --steps 10" "--virtual-ranks 8 --steps 3"; do
  echo "== tournament $w"
  timeout 300 python bench.py --workload tournament $w --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
done
for env in "GB_PASS_AHEAD=0" "GB_PASS_AHEAD=1"; do
  echo "== c2 $env"
  env $env timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['roofline']['frac'], d['e2e']['value']/1e9)"
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:train_pool_kernel.*Li1EE -s 2 -c 1 -o gpurun_out/pool_roll python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1
ls gpurun_out
