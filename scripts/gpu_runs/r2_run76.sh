# round 2, run 76: the --gpus N code path under torchrun with the NCCL backend
# at world size 1 (the sharded C3 workload forced; collectives over NCCL)
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 1 --workload c3shard --steps 3 --warmup 3 > gpurun_out/r2_76_nccl_w1.json 2> gpurun_out/r2_76_nccl_w1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 1 --workload c3shard --impl reference --steps 3 --warmup 3 > gpurun_out/r2_76_nccl_w1_ref.json 2> gpurun_out/r2_76_nccl_w1_ref.err
