# Evaluator: logistic regression on an 8-CTA cluster (DSMEM gradient
# reduction, one cluster barrier per step) vs the single-CTA kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for env in "GB_LOGREG_CLUSTER=0" "GB_LOGREG_CLUSTER=1"; do
  echo "== $env"
  env $env N=2000000 D=128 EPOCHS=10 timeout 600 python scripts/bench_logreg.py 2>&1 | tail -1
  env $env N=400000 D=32 EPOCHS=10 timeout 600 python scripts/bench_logreg.py 2>&1 | tail -1
done
