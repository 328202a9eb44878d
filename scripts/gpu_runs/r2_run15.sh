# round 2, run 15: practical ceiling of the pass's memory pattern (probe),
# where the C3 end-to-end embed time goes, ncu --set full of the pass kernel
# and the pair kernel at HEAD
mkdir -p gpurun_out
timeout 300 build/probe_rows > gpurun_out/r2_15_probe_rows.jsonl 2>&1
timeout 600 python scripts/profile_multilevel_e2e.py > gpurun_out/r2_15_e2e_phases.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_passes_kernel --launch-skip 6 -c 1 -f -o gpurun_out/r2_15_pass python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-multilevel > gpurun_out/r2_15_pass_ncu.log 2>&1
GB_ROTATION_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_pool_kernel --launch-skip 8 -c 1 -f -o gpurun_out/r2_15_pair python bench.py --workload tournament --virtual-ranks 1 --rotations 2 --steps 3 --warmup 3 > gpurun_out/r2_15_pair_ncu.log 2>&1
