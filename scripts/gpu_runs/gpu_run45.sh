# Small-level (latency variant) profile: V=2128 dense level, caps 256/590;
# lane layouts; one ncu capture at cap 256.
mkdir -p gpurun_out
for l in 8 16 32; do
  GB_GROUP_LANES=$l CAPS=256,590 timeout 300 python scripts/profile_small_level.py 2>/dev/null
done
CAPS=256 NCU=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:train_passes_kernel -s 1 -c 1 -o gpurun_out/small_lat python scripts/profile_small_level.py > /dev/null 2>&1
ls gpurun_out
