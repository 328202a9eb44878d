# round 2, run 9: CUDA-graph rotations with the bare capture API (graph on/off,
# K=16 x3, K=2, d=256), C3 embed time at equal AUCROC (ours vs the oracle port
# on the host cores, full runs), C4-shape AUCROC on one GPU
mkdir -p gpurun_out
free -g > gpurun_out/r2_09_host.txt; nproc >> gpurun_out/r2_09_host.txt
timeout 600 python -m pytest tests/test_tournament.py -q -m gpu > gpurun_out/r2_09_tests.txt 2>&1
for i in 1 2 3; do for gr in 1 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 20 --warmup 3 > gpurun_out/r2_09_t16_${i}_$gr.json 2>gpurun_out/r2_09_t16_${i}_$gr.err
done; done
for gr in 1 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 1 --steps 20 --warmup 3 > gpurun_out/r2_09_t2_$gr.json 2>&1
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --dim 256 --steps 10 --warmup 3 > gpurun_out/r2_09_t16d256_$gr.json 2>&1
done
timeout 900 python scripts/c3_equal_auc.py > gpurun_out/r2_09_c3_equal_auc.jsonl 2> gpurun_out/r2_09_c3_equal_auc.err
RUNS=vertex,edge timeout 900 python scripts/c4_aucroc.py > gpurun_out/r2_09_c4_aucroc.jsonl 2> gpurun_out/r2_09_c4_aucroc.err
