# round 2, run 84: compute-sanitizer memcheck + racecheck on the row-block
# builds (per-row cursors, split hubs, kept R-MAT samples) and the tournament
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 0 python -m pytest tests/test_config_scale.py -q -m gpu -x -k "blocked or c5_path" > gpurun_out/r2_84_memcheck.txt 2>&1
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_tournament.py -q -m gpu -x -k "rotation_graph_deterministic or cache_keyed" > gpurun_out/r2_84_memcheck_tn.txt 2>&1
