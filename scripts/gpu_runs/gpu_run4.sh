mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
LANES=8,32 timeout 300 python scripts/sweep_layout.py 2>&1 | tail -4
FLAGS=0 LANES=8 timeout 300 python scripts/sweep_layout.py 2>&1 | tail -2
timeout 300 python scripts/bench_multilevel.py c1 1000 2>&1 | tail -7
GB_PIPE=0 timeout 300 python scripts/bench_multilevel.py c1 1000 2>&1 | tail -1
GB_GROUP_LANES=32 timeout 300 python scripts/bench_multilevel.py c1 1000 2>&1 | tail -1
timeout 900 python scripts/bench_multilevel.py c3 200 2>&1 | tail -7
