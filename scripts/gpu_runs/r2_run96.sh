# round 2, run 96: fp64 sigmoid on the group's lane 0 only (broadcast) --
# GPU suite, C2 pass, tournament K=2 / K=16
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r2_96_pytest.txt 2>&1
timeout 900 python bench.py --no-multilevel --no-cpu-baseline > gpurun_out/r2_96_bench.json 2> gpurun_out/r2_96_bench.err
for vr in 1 8; do timeout 600 python bench.py --workload tournament --virtual-ranks $vr --steps 10 --warmup 3 > gpurun_out/r2_96_t$vr.json 2>> gpurun_out/r2_96_t.err; done
