# round 2, run 27: C5 on one GPU -- d=256 pass over the finest level, then the
# full multilevel embed at d=256 (coarse levels released as the ladder descends)
mkdir -p gpurun_out
DIM=256 timeout 1200 python scripts/c5_shape.py > gpurun_out/r2_27_c5_shape_d256.jsonl 2> gpurun_out/r2_27_c5_shape_d256.err
timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_27_c5_multilevel.jsonl 2> gpurun_out/r2_27_c5_multilevel.err
