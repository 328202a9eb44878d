# Inline index chain (KIND 0) back as the default: tests, smoke, C2 line,
# launch list + ncu of the pass kernel, C3 edge-scaled ladder.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2>/dev/null; cat gpurun_out/bench_c2.json | cut -c1-200
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes_kernel -s 3 -c 1 -o gpurun_out/pass_k0 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
UNIT=edge-scaled timeout 1200 python scripts/bench_multilevel.py c3 1000 > gpurun_out/ml_c3_es.jsonl 2>/dev/null; grep -E '"level"|summary' gpurun_out/ml_c3_es.jsonl | cut -c1-200
ls gpurun_out
