# round 2, run 93: coarsen_all releases its sort workspace -- C5 end to end
# under the native allocator (twice), and under cudaMallocAsync (once)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_config_scale.py -q -m gpu -x -k "blocked or c5_path" > gpurun_out/r2_93_pytest.txt 2>&1
for i in 1 2; do PYTORCH_CUDA_ALLOC_CONF=backend:native timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_93_c5_native_$i.jsonl 2>> gpurun_out/r2_93.err; done
timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_93_c5_async.jsonl 2>> gpurun_out/r2_93.err
