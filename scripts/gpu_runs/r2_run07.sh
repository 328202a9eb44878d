# round 2, run 7: CUDA-graph rotations (device seed/lr table, *_dp kernels):
# tests, then the K=16 virtual-rank tournament with and without the graph
# (3 repeats x 20 steps of 8 rotations), K=2 and d=256 for reference; fixed
# I/O + CAS tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tournament.py tests/test_io.py tests/test_collapse_cas.py -q -m gpu > gpurun_out/r2_07_tests.txt 2>&1
for i in 1 2 3; do for gr in 1 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 20 --warmup 3 > gpurun_out/r2_07_t16_${i}_$gr.json 2>gpurun_out/r2_07_t16_${i}_$gr.err
python -c "import json; d=json.load(open('gpurun_out/r2_07_t16_${i}_$gr.json')); print(json.dumps({'rep':$i,'K':16,'dim':128,'graph':'$gr','value':d['value'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step'],'clocks':d['clocks']}))" >> gpurun_out/r2_07_t16.jsonl
done; done
for gr in 1 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 1 --steps 20 --warmup 3 > gpurun_out/r2_07_t2_$gr.json 2>&1
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --dim 256 --steps 10 --warmup 3 > gpurun_out/r2_07_t16d256_$gr.json 2>&1
done
