for P in 0 1; do
  FSX_TMA_COPYONLY=1 FSX_TMA_PERSIST=$P timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab8_plain$P.log 2>&1 && FSX_TMA_COPYONLY=1 FSX_TMA_PERSIST=$P timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ab8_launches$P.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab8_ncu$P.log 2>&1
done
