# round 2, run 1: source-row delta reductions vs plain stores -- C1 AUCROC over
# 30 seeds (paired with the reference's 30) for several in-flight policies, the
# GPU test suite, and the C2 bench for both builds
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_01_gpu.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2_01_pytest.txt 2>&1
for lib in delta store; do
  if [ $lib = store ]; then export GB_LIB_PATH=$PWD/build/ab_store/libgosh_b200.so; else unset GB_LIB_PATH; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_01_bench_$lib.json 2> gpurun_out/r2_01_bench_$lib.err
  SEEDS=1-30 POLICY="256/16;64/16;256/64;1024/4" TAG=$lib timeout 1500 python scripts/c1_auc_sweep.py >> gpurun_out/r2_01_c1_auc.jsonl 2> gpurun_out/r2_01_c1_$lib.err
done
