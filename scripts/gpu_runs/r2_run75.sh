# round 2, run 75: reserve_device_memory -- its test, then C5 end to end with
# HBM mapped once up front (twice) and without (once)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_memory.py -q -m gpu > gpurun_out/r2_75_pytest.txt 2>&1
for i in 1 2; do timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_75_c5_reserve_$i.jsonl 2>> gpurun_out/r2_75.err; done
RESERVE=0 timeout 1500 python scripts/c5_multilevel.py > gpurun_out/r2_75_c5_noreserve.jsonl 2>> gpurun_out/r2_75.err
