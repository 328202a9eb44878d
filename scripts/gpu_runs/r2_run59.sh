# round 2, run 59: launch list of the default bench and ncu --set full of the
# headline kernel at HEAD (the fp64-sigmoid HOT KIND 3 pass, default since
# commit 15910c2; the earlier captures were of the fp32-sigmoid instantiation)
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2_59_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_59_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_passes_kernel --launch-skip 4 -c 1 -f -o gpurun_out/r2_59_pass python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-multilevel > gpurun_out/r2_59_pass_ncu.log 2>&1
