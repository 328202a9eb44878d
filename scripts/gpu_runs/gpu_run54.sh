# Evaluator: logreg epoch with the next step's rows gathered during the
# gradient reduction (one gather round per 256-row step) -- tests + A/B.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for env in "GB_LIB_PATH=build/exp/libgosh_b200_evalold.so" "X=0"; do
  echo "== $env"
  env $env N=2000000 D=128 EPOCHS=10 timeout 600 python scripts/bench_logreg.py 2>&1 | tail -1
  env $env N=400000 D=32 EPOCHS=10 timeout 600 python scripts/bench_logreg.py 2>&1 | tail -1
done
