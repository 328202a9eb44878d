# round 2, run 60: fp64 sigmoid as the pair kernels' default too -- GPU suite,
# default bench (sharded C3 field), tournament K=2 / K=16 with both sigmoids
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r2_60_pytest.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2_60_bench.json 2> gpurun_out/r2_60_bench.err
for vr in 1 8; do
for fs in "" 1; do
GB_FAST_SIGMOID=$fs timeout 600 python bench.py --workload tournament --virtual-ranks $vr --steps 10 --warmup 3 > gpurun_out/r2_60_t${vr}_fs${fs:-auto}.json 2>> gpurun_out/r2_60_t.err
done; done
