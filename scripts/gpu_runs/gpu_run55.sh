# Evaluator: logreg rows in independent sub-batches (dots, butterflies and
# sigmoids interleaved) on top of the gather/reduction overlap.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
N=2000000 D=128 EPOCHS=10 timeout 600 python scripts/bench_logreg.py 2>&1 | tail -1
N=400000 D=32 EPOCHS=10 timeout 600 python scripts/bench_logreg.py 2>&1 | tail -1
