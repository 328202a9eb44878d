mkdir -p gpurun_out
CAPS=64 NCU=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes -s 1 -c 1 -o gpurun_out/prof_small2 python scripts/profile_small_level.py > /dev/null 2>&1; echo ncu $?
