# round 2, run 3: parts-only tournament (PartStore, host-staged parts), new
# bench fields (sharded C3 anchor), C1 AUCROC over 60 paired seeds for the
# default and the uncapped in-flight policy
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/r2_03_gpu.txt; free -g >> gpurun_out/r2_03_gpu.txt; nproc >> gpurun_out/r2_03_gpu.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2_03_pytest.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_03_bench.json 2> gpurun_out/r2_03_bench.err
SEEDS=1-60 POLICY="256/16;4096/1" TAG=delta_smem_60 timeout 1500 python scripts/c1_auc_sweep.py >> gpurun_out/r2_03_c1_auc.jsonl 2> gpurun_out/r2_03_c1.err
