mkdir -p gpurun_out
for lanes in 8 16 32; do GB_GROUP_LANES=$lanes CAPS=64,256,1024 PASSES=200 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -3; done
CAPS=256 PASSES=200 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -1
CAPS=256 NCU=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes -s 1 -c 1 -o gpurun_out/prof_small256 python scripts/profile_small_level.py > /dev/null 2>&1; echo ncu1 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_pool -s 6 -c 1 -o gpurun_out/prof_pool3 python bench.py --workload tournament --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu2 $?
