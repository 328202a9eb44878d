# round 2, run 101: large downloads into fresh numpy pages, with and without
# MADV_POPULATE_WRITE first
mkdir -p gpurun_out
timeout 600 python scripts/probe_download_populate.py > gpurun_out/r2_101_download.jsonl 2> gpurun_out/r2_101.err
