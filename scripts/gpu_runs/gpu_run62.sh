# Staged pass (KIND 3) as the default for uncapped launches: tests, smoke,
# C2 line, launch list + ncu of the staged kernel, C3 ladder; then the
# pair kernel with staged rows (-DGB_POOL_STAGED build) A/B (gpu_run63.sh).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2>/dev/null; cut -c1-160 gpurun_out/bench_c2.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes_kernel -s 3 -c 1 -o gpurun_out/pass_k3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
UNIT=edge-scaled timeout 1200 python scripts/bench_multilevel.py c3 1000 > gpurun_out/ml_c3_es.jsonl 2>/dev/null; grep -E '"level"|summary' gpurun_out/ml_c3_es.jsonl | cut -c1-200
SCALE=27 SAMPLES=1900000000 timeout 1500 python scripts/big_graph.py > gpurun_out/big27.jsonl 2>&1; grep '"pass"' gpurun_out/big27.jsonl | cut -c1-300
ls gpurun_out
mkdir -p gpurun_out
GB_LIB_PATH=build/exp/libgosh_b200_poolstaged.so timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for env in "X=0" "GB_LIB_PATH=build/exp/libgosh_b200_poolstaged.so" "X=0" "GB_LIB_PATH=build/exp/libgosh_b200_poolstaged.so"; do
  env $env timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env d128', d['value']/1e9, d['roofline']['frac'])"
  env $env timeout 300 python bench.py --workload tournament --dim 256 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env d256', d['value']/1e9, d['roofline']['frac'])"
done
