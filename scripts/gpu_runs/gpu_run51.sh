# Bit-exact coarsening at scale: device hierarchy vs the CPU oracle's
# sequential coarsen_all (C3 shape with the CSR build too; scale 24).
mkdir -p gpurun_out
SCALE=22 SAMPLES=126000000 CSR=1 timeout 1500 python scripts/coarsen_parity_big.py > gpurun_out/coarsen_parity.jsonl 2> gpurun_out/coarsen_parity.err; tail -2 gpurun_out/coarsen_parity.err
SCALE=24 SAMPLES=400000000 timeout 1800 python scripts/coarsen_parity_big.py >> gpurun_out/coarsen_parity.jsonl 2>> gpurun_out/coarsen_parity.err; tail -2 gpurun_out/coarsen_parity.err
cat gpurun_out/coarsen_parity.jsonl
