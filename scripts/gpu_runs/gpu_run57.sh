# Capped mid-size launches spread over all SMs (GB_SPREAD) -- C3-L2-like
# level (V=63K, ~1.4K avg degree, cap 3941) and the C3 ladder.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for env in "GB_SPREAD=0" "GB_SPREAD=1"; do
  env $env V=63056 P=0.023 CAPS=3941,2000 PASSES=100 timeout 300 python scripts/profile_small_level.py 2>/dev/null
done
for env in "GB_SPREAD=0" "GB_SPREAD=1"; do
  env $env UNIT=edge-scaled timeout 1200 python scripts/bench_multilevel.py c3 1000 2>/dev/null | grep -E '"level"|summary' | cut -c1-200
done
