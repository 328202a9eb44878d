mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tournament.py tests/test_gpu_parity.py -q -m gpu -x -k "tournament or virtual" 2>&1 | tail -3
timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 5 --warmup 3 > gpurun_out/bench_tour_k16.json 2>gpurun_out/bench_tour_k16.err; cat gpurun_out/bench_tour_k16.json
timeout 300 python bench.py --workload tournament --virtual-ranks 2 --steps 5 --warmup 3 > gpurun_out/bench_tour_k4.json 2>gpurun_out/bench_tour_k4.err; cat gpurun_out/bench_tour_k4.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/tour_k16_launches.csv python bench.py --workload tournament --virtual-ranks 8 --steps 1 --warmup 3 > /dev/null 2>&1; wc -l gpurun_out/tour_k16_launches.csv
