# round 2, run 71: C5 end to end with 2^31-key row blocks (half as many blocks)
mkdir -p gpurun_out
BLOCK_KEYS=2147483648 timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_71_c5_multilevel_b31.jsonl 2> gpurun_out/r2_71.err
timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_71_c5_multilevel_b30.jsonl 2>> gpurun_out/r2_71.err
