# Experiment: pass kernel with sample rows staged in shared memory by
# cp.async (KIND 3, GB_PASS_SMEM=1: 80 registers, 3 blocks/SM).
mkdir -p gpurun_out
GB_PASS_SMEM=1 timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for env in "GB_PASS_SMEM=0" "GB_PASS_SMEM=1" "GB_PASS_SMEM=0" "GB_PASS_SMEM=1"; do
  env $env timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env c2', d['value']/1e9, d['roofline']['frac'])"
done
GB_PASS_SMEM=1 UNIT=edge-scaled timeout 1200 python scripts/bench_multilevel.py c3 1000 2>/dev/null | grep -E '"level"|summary' | cut -c1-200
