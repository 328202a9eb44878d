mkdir -p gpurun_out
for vr in 4 8; do for vs in 0 auto; do
GB_VIRTUAL_STREAMS=$vs timeout 300 python bench.py --workload tournament --dim 256 --virtual-ranks $vr --steps 5 --warmup 3 > gpurun_out/t256_vr${vr}_$vs.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/t256_vr${vr}_$vs.json')); print(json.dumps({'dim':256,'virtual_ranks':$vr,'GB_VIRTUAL_STREAMS':'$vs','value':d['value'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step']}))"
done; done
