# round 2, run 31: fp64-sigmoid HOT instantiations (all pass kinds + pair
# kernels) vs the fp32 sigmoid: C2 pass, C3 edge-scaled ladder, tournament
# K=2 / K=16, d=256; GPU tests with the fp64 default
mkdir -p gpurun_out
GB_FAST_SIGMOID=0 timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2_31_pytest_f64.txt 2>&1
for i in 1 2; do for fs in 0 1; do
GB_FAST_SIGMOID=$fs timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-multilevel > gpurun_out/r2_31_c2_fs${fs}_$i.json 2>/dev/null
GB_FAST_SIGMOID=$fs timeout 300 python bench.py --workload tournament --virtual-ranks 1 --steps 8 --warmup 3 > gpurun_out/r2_31_t2_fs${fs}_$i.json 2>/dev/null
GB_FAST_SIGMOID=$fs timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 8 --warmup 3 > gpurun_out/r2_31_t16_fs${fs}_$i.json 2>/dev/null
GB_FAST_SIGMOID=$fs timeout 300 python bench.py --workload tournament --virtual-ranks 1 --dim 256 --steps 6 --warmup 3 > gpurun_out/r2_31_t2d256_fs${fs}_$i.json 2>/dev/null
done; done
for fs in 0 1; do
GB_FAST_SIGMOID=$fs UNIT=edge-scaled timeout 600 python scripts/bench_multilevel.py c3 1000 > gpurun_out/r2_31_c3_edge_fs$fs.jsonl 2>&1
done
