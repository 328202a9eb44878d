# round 2, run 62: coarsening phase breakdown on a half-C4 R-MAT, plain and
# under an ncu launch list
mkdir -p gpurun_out
SCALE=26 SAMPLES=1000000000 timeout 600 python scripts/profile_coarsen.py > gpurun_out/r2_62_coarsen_phases.jsonl 2> gpurun_out/r2_62.err
SCALE=26 SAMPLES=1000000000 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r2_62_launches.csv python scripts/profile_coarsen.py > gpurun_out/r2_62_ncu.log 2>&1
