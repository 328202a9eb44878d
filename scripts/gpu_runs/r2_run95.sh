# round 2, run 95: C5 scripts with max_split_size_mb=1024 as their default (twice);
# c5_shape (passes at d=128/256) once
mkdir -p gpurun_out
for i in 1 2; do timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_95_c5_$i.jsonl 2>> gpurun_out/r2_95.err; done
timeout 1500 python scripts/c5_shape.py > gpurun_out/r2_95_c5_shape.jsonl 2>> gpurun_out/r2_95.err
