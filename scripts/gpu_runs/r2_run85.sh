# round 2, run 85: C4-shape embed wall-time through train_multilevel(host graph) -> numpy
mkdir -p gpurun_out
timeout 1500 python scripts/c4_e2e.py > gpurun_out/r2_85_c4_e2e.jsonl 2> gpurun_out/r2_85.err
