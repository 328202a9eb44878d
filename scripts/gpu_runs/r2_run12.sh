# round 2, run 12: tournament K=16 with 32 rotations per step (graph auto vs
# off, 3 repeats), K=2 / d=256; ncu --set full of the C3 L3/L4 training
# launches; C4-shape coarsening parity against the oracle on the host
mkdir -p gpurun_out
for i in 1 2 3; do for gr in auto 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 8 --warmup 3 > gpurun_out/r2_12_t16_${i}_$gr.json 2>gpurun_out/r2_12_t16_${i}_$gr.err
done; done
for gr in auto 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 1 --steps 8 --warmup 3 > gpurun_out/r2_12_t2_$gr.json 2>&1
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --dim 256 --steps 4 --warmup 3 > gpurun_out/r2_12_t16d256_$gr.json 2>&1
done
for L in 4 3; do
LEVEL=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes -c 1 -f -o gpurun_out/r2_12_c3_L$L python scripts/profile_c3_levels.py > gpurun_out/r2_12_c3_L$L.log 2>&1
LEVEL=$L timeout 300 python scripts/profile_c3_levels.py >> gpurun_out/r2_12_c3_levels_plain.jsonl 2>&1
done
timeout 3300 python scripts/c4_coarsen_parity.py > gpurun_out/r2_12_c4_coarsen.jsonl 2> gpurun_out/r2_12_c4_coarsen.err
