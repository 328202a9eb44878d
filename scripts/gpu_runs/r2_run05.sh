# round 2, run 5 (re-entry): GPU suite at HEAD, default bench + reference arm,
# launch list of the bench, C3 edge-scaled ladder and C3 AUCROC for the
# uncapped (new default) vs max(256, V/16) in-flight policy
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2_05_gpu.txt; nproc >> gpurun_out/r2_05_gpu.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_05_pytest.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_05_bench.json 2> gpurun_out/r2_05_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_05_bench_ref.json 2> gpurun_out/r2_05_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_05_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_05_ncu_bench.log 2>&1
UNIT=edge-scaled timeout 600 python scripts/bench_multilevel.py c3 1000 > gpurun_out/r2_05_c3_edge_uncapped.jsonl 2>&1
GB_INFLIGHT_FLOOR=256 GB_INFLIGHT_DIV=16 UNIT=edge-scaled timeout 600 python scripts/bench_multilevel.py c3 1000 > gpurun_out/r2_05_c3_edge_capped.jsonl 2>&1
for pol in "4096 1" "256 16"; do set -- $pol
GB_INFLIGHT_FLOOR=$1 GB_INFLIGHT_DIV=$2 GRAPH=c3 MODES=cap0 SEEDS=1,2,3 UNIT=vertex-pass EPOCHS=1000 EVAL_SAMPLE=1000000 timeout 900 python scripts/auc_modes.py >> gpurun_out/r2_05_c3_auc_policy_$1_$2.jsonl 2>&1
done
