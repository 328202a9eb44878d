# round 2, run 65: kernel launch list of the C5-shape coarsening (row-block builds)
mkdir -p gpurun_out
SCALE=28 SAMPLES=4300000000 BLOCK=1073741824 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r2_65_launches.csv python scripts/profile_coarsen.py > gpurun_out/r2_65.log 2>&1
