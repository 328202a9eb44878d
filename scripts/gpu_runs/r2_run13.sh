# round 2, run 13: cached rotation graphs, spread tiny-level launches
# (GB_SPREAD A/B on the C3 ladders), C4-shape coarsening test, how many levels
# to shard on C3 (AUCROC + projected 8-GPU time)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_tournament.py tests/test_config_scale.py -q -m gpu > gpurun_out/r2_13_tests.txt 2>&1
for sp in 1 0; do
GB_SPREAD=$sp UNIT=edge-scaled timeout 600 python scripts/bench_multilevel.py c3 1000 > gpurun_out/r2_13_c3_edge_spread$sp.jsonl 2>&1
GB_SPREAD=$sp UNIT=vertex-pass timeout 600 python scripts/bench_multilevel.py c3 1000 > gpurun_out/r2_13_c3_vertex_spread$sp.jsonl 2>&1
done
for i in 1 2 3; do for gr in auto 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 8 --warmup 3 > gpurun_out/r2_13_t16_${i}_$gr.json 2>gpurun_out/r2_13_t16_${i}_$gr.err
done; done
for gr in auto 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 1 --steps 8 --warmup 3 > gpurun_out/r2_13_t2_$gr.json 2>&1
done
RANKS=8 SHARD=1,2,3 timeout 1500 python scripts/c3_shard_levels.py > gpurun_out/r2_13_c3_shard_levels.jsonl 2> gpurun_out/r2_13_c3_shard_levels.err
