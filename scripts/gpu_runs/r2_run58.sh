# round 2, run 58: HEAD re-check of the --gpus N bench path (torchrun, 2 and
# 4 ranks sharing the one GPU over gloo); numbers are meaningless here
mkdir -p gpurun_out
for n in 2 4; do
GB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --steps 3 --warmup 3 > gpurun_out/r2_58_torchrun_$n.json 2> gpurun_out/r2_58_torchrun_$n.err
GB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --impl reference --gpus $n --steps 3 --warmup 3 > gpurun_out/r2_58_torchrun_ref_$n.json 2> gpurun_out/r2_58_torchrun_ref_$n.err
done
