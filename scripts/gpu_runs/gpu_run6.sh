mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
CAPS=16,64,256 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -3
GB_GROUP_LANES=8 CAPS=64 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -1
DIM=32 CAPS=64 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -1
timeout 300 python scripts/bench_multilevel.py c1 1000 2>&1 | tail -1
timeout 900 python scripts/bench_multilevel.py c3 200 2>&1 | tail -6
CAPS=0 SEEDS=1,2,3,4,5 timeout 900 python scripts/c1_gpu_auc.py 2>&1 | tail -1
