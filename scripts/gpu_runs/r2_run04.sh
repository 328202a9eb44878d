# round 2, run 4: GPU suite (host-staged parts fix, blocked CSR / coarsening,
# C5 budget path), uncapped default: C3 edge-scaled ladder timing and C3
# AUCROC of the old (256/16) vs new (uncapped) in-flight policy
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_04_pytest.txt 2>&1
UNIT=edge-scaled timeout 600 python scripts/bench_multilevel.py c3 1000 > gpurun_out/r2_04_c3_edge_uncapped.jsonl 2>&1
GB_INFLIGHT_FLOOR=256 GB_INFLIGHT_DIV=16 UNIT=edge-scaled timeout 600 python scripts/bench_multilevel.py c3 1000 > gpurun_out/r2_04_c3_edge_capped.jsonl 2>&1
for pol in "4096 1" "256 16"; do set -- $pol
GB_INFLIGHT_FLOOR=$1 GB_INFLIGHT_DIV=$2 GRAPH=c3 MODES=cap0 SEEDS=1,2,3 UNIT=vertex-pass EPOCHS=1000 EVAL_SAMPLE=1000000 timeout 900 python scripts/auc_modes.py >> gpurun_out/r2_04_c3_auc_policy_$1_$2.jsonl 2>&1
done
