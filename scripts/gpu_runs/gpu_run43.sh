# HEAD check: tests, smoke, C2 bench line, tournament K=2.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 400 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2>/dev/null; cat gpurun_out/bench_c2.json
timeout 300 python bench.py --workload tournament --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tournament', d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes_kernel -s 3 -c 1 -o gpurun_out/pass_k2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
