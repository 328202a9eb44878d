mkdir -p gpurun_out
for i in 1 2 3; do for vs in 1 0; do
GB_VIRTUAL_STREAMS=$vs timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 5 --warmup 3 > gpurun_out/trep_${i}_$vs.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/trep_${i}_$vs.json')); print(json.dumps({'rep':$i,'dim':128,'virtual_ranks':8,'GB_VIRTUAL_STREAMS':'$vs','value':d['value'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step'],'clocks':d['clocks']}))" | tee -a gpurun_out/trep.jsonl
done; done
GB_VIRTUAL_STREAMS=1 timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('long', d['value']/1e9, d['ms_per_step'])"
