# C2 pass: index chain one source ahead (KIND 2, GB_PASS_AHEAD=1) A/B; GPU
# tests under both settings.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
GB_PASS_AHEAD=1 timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for env in "GB_PASS_AHEAD=0" "GB_PASS_AHEAD=1" "GB_PASS_AHEAD=0" "GB_PASS_AHEAD=1"; do
  echo "== c2 $env"
  env $env timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['roofline']['frac'], d['e2e']['value']/1e9)"
done
GB_PASS_AHEAD=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes_kernel -s 5 -c 1 -o gpurun_out/pass_ahead python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
