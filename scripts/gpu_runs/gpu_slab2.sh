# slab bench path at world size 1: fused p2p exchange (auto) vs NCCL, and 3D
for X in auto nccl; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --slab --exchange $X --config cfg2 --steps 5 --warmup 3 > gpurun_out/slab2_cfg2_$X.log 2>&1; tail -c 1600 gpurun_out/slab2_cfg2_$X.log; echo
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29542 bench.py --slab --config cfg4 --steps 3 --warmup 3 > gpurun_out/slab2_cfg4.log 2>&1; tail -c 600 gpurun_out/slab2_cfg4.log
