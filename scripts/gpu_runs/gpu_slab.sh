timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_slab.log 2>&1; tail -3 gpurun_out/pytest_slab.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --slab --config cfg3 --steps 3 --warmup 3 > gpurun_out/bench_slab_cfg3.log 2>&1; tail -c 1500 gpurun_out/bench_slab_cfg3.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -c 1200 gpurun_out/bench_ref.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; tail -c 2500 gpurun_out/bench_full.log
nproc; free -g | head -2; lscpu | grep "Model name"
