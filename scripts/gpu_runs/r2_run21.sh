# round 2, run 21: C3 coarse levels, latency variant (GB_PIPE=1) vs default
mkdir -p gpurun_out
for L in 4 3 2; do for pipe in default 1 0; do
if [ $pipe = default ]; then unset GB_PIPE; else export GB_PIPE=$pipe; fi
LEVEL=$L EPOCHS=40 timeout 300 python scripts/profile_c3_levels.py >> gpurun_out/r2_21_levels.jsonl 2>&1
done; done
