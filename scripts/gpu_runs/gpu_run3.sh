set -x
mkdir -p gpurun_out
timeout 900 python scripts/bench_multilevel.py c3 1000 2>&1 | tail -20
timeout 300 python scripts/bench_multilevel.py c1 1000 2>&1 | tail -10
CAPS=0,64 SEEDS=1,2,3,4,5 timeout 900 python scripts/c1_gpu_auc.py 2>&1 | tail -3
