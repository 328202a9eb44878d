# round 2, run 61: pair kernel with 16 lanes per source (VecRow<16,2>, half the
# row registers) vs the default 8, K=2 and K=16; the rotation-graph cache test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tournament.py -q -m gpu -x > gpurun_out/r2_61_pytest.txt 2>&1
for vr in 1 8; do
for lanes in "" 16; do
GB_GROUP_LANES=$lanes timeout 600 python bench.py --workload tournament --virtual-ranks $vr --steps 10 --warmup 3 > gpurun_out/r2_61_t${vr}_g${lanes:-8}.json 2>> gpurun_out/r2_61_t.err
done; done
