timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/slab3_launch_p2p.csv python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29543 bench.py --slab --exchange p2p --config cfg2 --steps 2 --warmup 3 > gpurun_out/slab3_ncu.log 2>&1
python scripts/launches.py gpurun_out/slab3_launch_p2p.csv
