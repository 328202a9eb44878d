# round 2, run 11: full GPU suite at HEAD, smoke, tournament K=16 with 32
# rotations per step (graph auto vs off, 3 repeats), K=2 / d=256
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_11_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_11_smoke.txt 2>&1
for i in 1 2 3; do for gr in auto 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 10 --warmup 2 > gpurun_out/r2_11_t16_${i}_$gr.json 2>gpurun_out/r2_11_t16_${i}_$gr.err
done; done
for gr in auto 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 1 --steps 10 --warmup 2 > gpurun_out/r2_11_t2_$gr.json 2>&1
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --dim 256 --steps 5 --warmup 2 > gpurun_out/r2_11_t16d256_$gr.json 2>&1
done
