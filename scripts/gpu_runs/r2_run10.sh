# round 2, run 10: graph-rotation phase timing (K=16 and K=2), C3 AUCROC vs
# concurrency: the reference path (oracle) with 1 and 16 host threads, the
# device path uncapped and capped
mkdir -p gpurun_out
VR=8 timeout 300 python scripts/rotation_graph_timing.py > gpurun_out/r2_10_rot_timing_k16.jsonl 2>&1
VR=1 timeout 300 python scripts/rotation_graph_timing.py > gpurun_out/r2_10_rot_timing_k2.jsonl 2>&1
MODES=gpu,gpu_cap16384,gpu_cap4096,gpu_cap1024,gpu_cap256,ref_w16,ref_w1 timeout 1500 python scripts/c3_concurrency_auc.py > gpurun_out/r2_10_c3_concurrency.jsonl 2> gpurun_out/r2_10_c3_concurrency.err
