# Refresh at HEAD: tests, smoke, C2 bench line (+ CPU leg), reference arm, C2
# launch list + ncu of the HOT pass kernel, C1 AUCROC (5 seeds, twice),
# C3 multilevel edge-scaled with per-level timings.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 400 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>/dev/null; cat gpurun_out/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes_kernel -s 8 -c 1 -o gpurun_out/pass_hot python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
CAPS=0 SEEDS=1,2,3,4,5 timeout 900 python scripts/c1_gpu_auc.py > gpurun_out/c1auc.jsonl 2>/dev/null; cat gpurun_out/c1auc.jsonl
CAPS=0 SEEDS=1,2,3,4,5 timeout 900 python scripts/c1_gpu_auc.py >> gpurun_out/c1auc.jsonl 2>/dev/null; tail -1 gpurun_out/c1auc.jsonl
UNIT=edge-scaled timeout 1200 python scripts/bench_multilevel.py c3 1000 > gpurun_out/ml_c3_es.jsonl 2>/dev/null; cat gpurun_out/ml_c3_es.jsonl | cut -c1-250
ls gpurun_out
