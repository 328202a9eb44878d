# Experiment: L1-cached row loads (ld.ca) -- parity tests and C2/tournament A/B.
mkdir -p gpurun_out
GB_LIB_PATH=build/exp/libgosh_b200_ldca.so timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for env in "X=0" "GB_LIB_PATH=build/exp/libgosh_b200_ldca.so" "X=0" "GB_LIB_PATH=build/exp/libgosh_b200_ldca.so"; do
  echo "== $env"
  env $env timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value']/1e9, d['roofline']['frac'])"
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tournament', d['value']/1e9, d['roofline']['frac'])"
done
# C3 edge-scaled (the finest level's budget is many rotations, no max(1, .) floor):
# in-memory vs tournament over 4 / 8 virtual ranks
GRAPH=c3 MODES=cap0,tour4,tour8 SEEDS=1 UNIT=edge-scaled EPOCHS=1000 EVAL_SAMPLE=1000000 timeout 2400 python scripts/auc_modes.py > gpurun_out/c3_auc_tour_es.jsonl 2> gpurun_out/c3_auc_tour_es.err; tail -2 gpurun_out/c3_auc_tour_es.err; cut -c1-300 gpurun_out/c3_auc_tour_es.jsonl
