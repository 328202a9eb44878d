# round 2, run 102: launch list of the default bench at HEAD (fp64-sigmoid pair
# kernels in the sharded field) and ncu --set full of the fp64 pair kernel
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2_102_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_102_launches.log 2>&1
GB_ROTATION_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_pool_kernel --launch-skip 8 -c 1 -f -o gpurun_out/r2_102_pair python bench.py --workload tournament --virtual-ranks 1 --rotations 2 --steps 3 --warmup 3 > gpurun_out/r2_102_pair_ncu.log 2>&1
