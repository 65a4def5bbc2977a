# slab path under torchrun (world 1, both exchanges) + cfg2 launch list without the spectral-cut steps
for x in p2p nccl; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29553 bench.py --gpus 1 --slab --exchange $x --config cfg2 --steps 5 --warmup 3 > gpurun_out/m_slab_$x.log 2>&1; python scripts/summarize.py gpurun_out/m_slab_$x.log; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01e_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cut > gpurun_out/m_ncu.log 2>&1
python scripts/launches.py gpurun_out/r01e_launches_cfg2.csv | tail -4
