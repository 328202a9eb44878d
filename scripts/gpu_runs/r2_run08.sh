# round 2, run 8: warp-uniform KIND 3 pass (A/B against the previous build),
# CUDA-graph tournament rotations K=16 (graph on/off, 3 repeats), new tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tournament.py tests/test_collapse_cas.py tests/test_config_scale.py tests/test_gpu_parity.py -q -m gpu > gpurun_out/r2_08_tests.txt 2>&1
for i in 1 2; do for lib in new old; do
  if [ $lib = old ]; then export GB_LIB_PATH=$PWD/build/ab_k3old/libgosh_b200.so; else unset GB_LIB_PATH; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-multilevel > gpurun_out/r2_08_c2_${lib}_$i.json 2> gpurun_out/r2_08_c2_${lib}_$i.err
done; done
unset GB_LIB_PATH
for i in 1 2 3; do for gr in 1 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --steps 20 --warmup 3 > gpurun_out/r2_08_t16_${i}_$gr.json 2>gpurun_out/r2_08_t16_${i}_$gr.err
done; done
for gr in 1 0; do
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 1 --steps 20 --warmup 3 > gpurun_out/r2_08_t2_$gr.json 2>&1
GB_ROTATION_GRAPH=$gr timeout 300 python bench.py --workload tournament --virtual-ranks 8 --dim 256 --steps 10 --warmup 3 > gpurun_out/r2_08_t16d256_$gr.json 2>&1
done
