# round 2, run 2: S0 kept in shared memory (KIND 0/2/3, pair kernels) -- C2
# bench cost of the source-row delta write-back, config-scale tests, C1 AUCROC
# for wider in-flight policies, the new bench fields
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2_02_pytest.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_02_bench.json 2> gpurun_out/r2_02_bench.err
SEEDS=1-30 POLICY="1024/4;1024/1;4096/1;256/4;100000000/1" TAG=delta_smem timeout 1500 python scripts/c1_auc_sweep.py >> gpurun_out/r2_02_c1_auc.jsonl 2> gpurun_out/r2_02_c1.err
