mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tournament.py tests/test_gpu_parity.py -q -m gpu -x -k "tournament or virtual" 2>&1 | tail -2
for dim in 128 256; do
timeout 300 python bench.py --workload tournament --dim $dim --virtual-ranks 8 --steps 5 --warmup 3 > gpurun_out/tauto_$dim.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/tauto_$dim.json')); print(json.dumps({'dim':$dim,'virtual_ranks':8,'GB_VIRTUAL_STREAMS':'auto (48 MiB rule)','value':d['value'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step']}))" | tee -a gpurun_out/tauto.jsonl
done
