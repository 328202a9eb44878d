mkdir -p gpurun_out
timeout 300 python scripts/profile_small_level.py 2>&1 | tail -6
GB_GROUP_LANES=32 CAPS=64,256 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -2
GB_PIPE=0 CAPS=64,256 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -2
DIM=32 CAPS=64 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -1
CAPS=64 NCU=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes -s 1 -c 1 -o gpurun_out/prof_small python scripts/profile_small_level.py > /dev/null 2>&1; echo ncu $?
