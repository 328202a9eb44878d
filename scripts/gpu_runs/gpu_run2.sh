set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python scripts/sweep_layout.py 2>&1 | tail -8
CAPS=0,1024,16384 LANES=8 timeout 300 python scripts/sweep_layout.py 2>&1 | tail -4
timeout 400 python bench.py --steps 30 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
CAPS=0,4096 SEEDS=1,2,3 timeout 900 python scripts/c1_gpu_auc.py 2>&1 | tail -5
timeout 400 ncu --set full --clock-control none --import-source on -k regex:train_passes -s 3 -c 1 -o gpurun_out/prof_train2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu $?
