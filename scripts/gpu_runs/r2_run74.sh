# round 2, run 74: allocation cost in the C5-shape coarsening -- default pool
# vs the pool's release threshold at max with 160 GiB mapped up front
mkdir -p gpurun_out
for i in 1 2; do
GB_TRACE_BLOCKS=1 SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_74_default_$i.jsonl 2>> gpurun_out/r2_74.err
RELEASE=1 WARM_GIB=160 GB_TRACE_BLOCKS=1 SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1200 python scripts/profile_coarsen.py > gpurun_out/r2_74_warm_$i.jsonl 2>> gpurun_out/r2_74.err
done
