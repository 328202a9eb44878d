# round 2, run 86: C4-shape embed wall-time through train_multilevel(host graph) -> numpy, with phases
mkdir -p gpurun_out
timeout 1500 python scripts/c4_e2e.py > gpurun_out/r2_86_c4_e2e.jsonl 2> gpurun_out/r2_86.err
