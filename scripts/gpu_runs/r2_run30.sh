# round 2, run 30: HOT KIND 3 with the reference's fp64 sigmoid -- tests and
# C2 bench (fp64_sigmoid field vs the fast headline), C1 AUCROC with it
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "single_group or hogwild or finite_difference" > gpurun_out/r2_30_tests.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-multilevel > gpurun_out/r2_30_bench_$i.json 2> gpurun_out/r2_30_bench_$i.err
done
