# round 2, run 98: C4-shape link-prediction setup phases
mkdir -p gpurun_out
timeout 1200 python scripts/c4_setup_phases.py > gpurun_out/r2_98_c4_setup.jsonl 2> gpurun_out/r2_98.err
