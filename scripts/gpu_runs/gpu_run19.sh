mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -4
DETERMINISTIC=1 CAPS=0 SEEDS=1 timeout 1200 python scripts/c1_gpu_auc.py > gpurun_out/c1auc_det2.jsonl 2>&1; tail -2 gpurun_out/c1auc_det2.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes -s 3 -c 1 -o gpurun_out/prof_train_atomic python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu2 $?
SCALE=27 SAMPLES=1900000000 timeout 1500 python scripts/big_graph.py > gpurun_out/big27.jsonl 2>&1; echo rc $?; tail -12 gpurun_out/big27.jsonl
