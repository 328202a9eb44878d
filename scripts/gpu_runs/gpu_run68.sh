mkdir -p gpurun_out
# virtual-rank tournament: one stream per virtual rank vs serialised
timeout 600 python -m pytest tests/test_tournament.py tests/test_gpu_parity.py -q -m gpu -x -k "tournament or virtual" 2>&1 | tail -5
for vr in 2 4 8; do
for env in GB_VIRTUAL_STREAMS=0 GB_VIRTUAL_STREAMS=1; do
  env $env timeout 300 python bench.py --workload tournament --virtual-ranks $vr --steps 5 --warmup 3 > gpurun_out/tour_vr${vr}_${env}.json 2>gpurun_out/tour_vr${vr}_${env}.err
  python -c "import json; d=json.load(open('gpurun_out/tour_vr${vr}_${env}.json')); print('vr=$vr $env', round(d['value']/1e9,3), 'G upd/s frac', round(d['roofline']['frac'],3), 'ms', round(d['ms_per_step'],2))"
done
done
