# Balanced pools: GPU tests, tournament throughput, C3 edge-scaled AUCROC of
# the balanced tournament (in-memory 0.826, reference-pool tournament 0.782/0.778).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tournament', d['value']/1e9, d['roofline']['frac'])"
GRAPH=c3 MODES=tour4b,tour8b SEEDS=1 UNIT=edge-scaled EPOCHS=1000 EVAL_SAMPLE=1000000 timeout 2400 python scripts/auc_modes.py > gpurun_out/c3_auc_bal_es.jsonl 2> gpurun_out/c3_auc_bal_es.err; tail -3 gpurun_out/c3_auc_bal_es.err; cut -c1-300 gpurun_out/c3_auc_bal_es.jsonl
