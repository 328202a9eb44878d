# round 2, run 20: staged pair kernels (80 registers, 3 blocks/SM) A/B --
# GPU suite with GB_POOL_STAGED=1, tournament K=2/K=16 at d=128 and d=256
mkdir -p gpurun_out
GB_POOL_STAGED=1 timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2_20_pytest_staged.txt 2>&1
for i in 1 2; do for st in 1 0; do
GB_POOL_STAGED=$st timeout 300 python bench.py --workload tournament --virtual-ranks 1 --steps 8 --warmup 3 > gpurun_out/r2_20_t2_${st}_$i.json 2>&1
GB_POOL_STAGED=$st timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 8 --warmup 3 > gpurun_out/r2_20_t16_${st}_$i.json 2>&1
GB_POOL_STAGED=$st timeout 300 python bench.py --workload tournament --virtual-ranks 1 --dim 256 --steps 6 --warmup 3 > gpurun_out/r2_20_t2d256_${st}_$i.json 2>&1
GB_POOL_STAGED=$st timeout 300 python bench.py --workload tournament --virtual-ranks 8 --dim 256 --steps 4 --warmup 3 > gpurun_out/r2_20_t16d256_${st}_$i.json 2>&1
done; done
